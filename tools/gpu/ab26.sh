for v in np4m8 np4m6; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_raster.py init $v >> gpurun_out/ab26.log 2>&1; done
