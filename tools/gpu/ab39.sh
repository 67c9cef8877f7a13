for v in base tf1 tf1b3 base tf1; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_raster.py init $v >> gpurun_out/ab40.log 2>&1; done
SALF_LIB=build_ab/base/libsalf_b200.so python tools/ab_raster.py surface base_s >> gpurun_out/ab40.log 2>&1
SALF_LIB=build_ab/tf1/libsalf_b200.so python tools/ab_raster.py surface tf1_s >> gpurun_out/ab40.log 2>&1
