python -m pytest tests -m gpu -x -q > gpurun_out/t37.log 2>&1; echo rc=$? >> gpurun_out/t37.log
python tools/ab_raster.py init rows > gpurun_out/ab27.log 2>&1
python tools/ab_raster.py surface rows_s >> gpurun_out/ab27.log 2>&1
