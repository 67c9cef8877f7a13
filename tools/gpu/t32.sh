python -m pytest tests -m gpu -x -q > gpurun_out/t32.log 2>&1; echo rc=$? >> gpurun_out/t32.log
python tools/ab_ray.py mixedbwd > gpurun_out/ab21.log 2>&1
python tools/prof_c5.py > gpurun_out/c5prof3.log 2>&1
