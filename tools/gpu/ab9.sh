python -m pytest tests -m gpu -x -q -k "backward or train or actors" > gpurun_out/t12.log 2>&1; echo rc=$? >> gpurun_out/t12.log
python tools/ab_raster.py init cur > gpurun_out/ab9.log 2>&1
