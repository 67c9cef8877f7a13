python -m pytest tests -m gpu -x -q -k "raster or certified or actors or train or density or tile" > gpurun_out/t41.log 2>&1; echo rc=$? >> gpurun_out/t41.log
python tools/ab_raster.py init order > gpurun_out/ab32.log 2>&1
SALF_TILE_ORDER=0 python tools/ab_raster.py init noorder >> gpurun_out/ab32.log 2>&1
python tools/ab_raster.py surface order_s >> gpurun_out/ab32.log 2>&1
SALF_TILE_ORDER=0 python tools/ab_raster.py surface noorder_s >> gpurun_out/ab32.log 2>&1
