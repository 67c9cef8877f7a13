python tools/ab_raster.py init ftz > gpurun_out/ab39.log 2>&1
python tools/ab_raster.py init ftz2 >> gpurun_out/ab39.log 2>&1
python tools/ab_raster.py surface ftz_s >> gpurun_out/ab39.log 2>&1
python tools/ab_ray.py ftz >> gpurun_out/ab39.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/t49.log 2>&1; echo rc=$? >> gpurun_out/t49.log
