timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t62.log 2>&1; echo rc=$? >> gpurun_out/t62.log
timeout 300 python tools/ab_ray.py depthonly >> gpurun_out/ab53.log 2>&1
