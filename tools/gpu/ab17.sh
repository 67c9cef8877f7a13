python -m pytest tests -m gpu -x -q -k "raster or certified or actors or train or density or effects or ray" > gpurun_out/t25.log 2>&1; echo rc=$? >> gpurun_out/t25.log
python tools/ab_raster.py init cur > gpurun_out/ab17.log 2>&1
python tools/ab_raster.py surface surf >> gpurun_out/ab17.log 2>&1
SALF_NO_REDO=1 python tools/ab_raster.py init noredo >> gpurun_out/ab17.log 2>&1
