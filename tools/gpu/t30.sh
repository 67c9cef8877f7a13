python -m pytest tests -m gpu -x -q > gpurun_out/t30.log 2>&1; echo rc=$? >> gpurun_out/t30.log
python tools/gpu/lid_time.py cert > gpurun_out/lid2.log 2>&1
python tools/ab_ray.py cert > gpurun_out/ab20.log 2>&1
