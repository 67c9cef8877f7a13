python -m pytest tests -m gpu -x -q -k "raster or certified or actors or train or density" > gpurun_out/t19.log 2>&1; echo rc=$? >> gpurun_out/t19.log
python tools/ab_raster.py init cur > gpurun_out/ab11.log 2>&1
SALF_NO_REDO=1 python tools/ab_raster.py init noredo >> gpurun_out/ab11.log 2>&1
SALF_NO_REDO=1 python tools/ab_raster.py surface surf_noredo >> gpurun_out/ab11.log 2>&1
