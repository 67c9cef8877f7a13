python -m pytest tests -m gpu -x -q -k "raster or certified or actors or train or density" > gpurun_out/t24.log 2>&1; echo rc=$? >> gpurun_out/t24.log
python tools/ab_raster.py init cur > gpurun_out/ab16.log 2>&1
