python tools/ab_raster.py init cur > gpurun_out/ab18.log 2>&1
for v in c128 c32 cb64 cb16; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_raster.py init $v >> gpurun_out/ab18.log 2>&1; done
