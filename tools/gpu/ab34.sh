python -m pytest tests -m gpu -x -q -k "raster or certified or actors or tile or stress" > gpurun_out/t43.log 2>&1; echo rc=$? >> gpurun_out/t43.log
python tools/ab_raster.py init async > gpurun_out/ab34.log 2>&1
SALF_LIB=build_ab/noasync/libsalf_b200.so python tools/ab_raster.py init noasync >> gpurun_out/ab34.log 2>&1
python tools/ab_raster.py surface async_s >> gpurun_out/ab34.log 2>&1
SALF_LIB=build_ab/noasync/libsalf_b200.so python tools/ab_raster.py surface noasync_s >> gpurun_out/ab34.log 2>&1
