python -m pytest tests -m gpu -x -q > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
python tools/ab_raster.py init cur > gpurun_out/ab8.log 2>&1
SALF_NO_REDO=1 python tools/ab_raster.py init noredo >> gpurun_out/ab8.log 2>&1
python tools/ab_raster.py surface surf >> gpurun_out/ab8.log 2>&1
SALF_NO_REDO=1 python tools/ab_raster.py surface surf_noredo >> gpurun_out/ab8.log 2>&1
