python -m pytest tests -m gpu -x -q -k "ray or lidar or c3 or c4 or stress or raw or effects" > gpurun_out/t40.log 2>&1; echo rc=$? >> gpurun_out/t40.log
python tools/ab_ray.py persist > gpurun_out/ab30.log 2>&1
python tools/gpu/lid_time.py persist >> gpurun_out/ab30.log 2>&1
