python -m pytest tests -m gpu -x -q -k "raster or certified or actors or train or density" > gpurun_out/t20.log 2>&1; echo rc=$? >> gpurun_out/t20.log
python tools/ab_raster.py init cur > gpurun_out/ab12.log 2>&1
python tools/ab_raster.py surface surf >> gpurun_out/ab12.log 2>&1
