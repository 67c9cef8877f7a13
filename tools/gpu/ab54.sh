for v in bm4 bm5 bm6 bm4 bm5; do SALF_LIB=build_ab/$v/libsalf_b200.so timeout 300 python tools/ab_raster.py init $v >> gpurun_out/ab54.log 2>&1; done
