python -m pytest tests -m gpu -x -q -k "raster or certified or tile or stress or backward" > gpurun_out/t48.log 2>&1; echo rc=$? >> gpurun_out/t48.log
SALF_LIB=build_ab/nofuse/libsalf_b200.so python tools/ab_raster.py init nofuse > gpurun_out/ab38.log 2>&1
SALF_LIB=build_ab/fuse/libsalf_b200.so python tools/ab_raster.py init fuse >> gpurun_out/ab38.log 2>&1
SALF_LIB=build_ab/nofuse/libsalf_b200.so python tools/ab_raster.py init nofuse2 >> gpurun_out/ab38.log 2>&1
SALF_LIB=build_ab/fuse/libsalf_b200.so python tools/ab_raster.py init fuse2 >> gpurun_out/ab38.log 2>&1
SALF_LIB=build_ab/nofuse/libsalf_b200.so python tools/ab_raster.py surface nofuse_s >> gpurun_out/ab38.log 2>&1
SALF_LIB=build_ab/fuse/libsalf_b200.so python tools/ab_raster.py surface fuse_s >> gpurun_out/ab38.log 2>&1
