python tools/ab_raster.py init pf > gpurun_out/ab31.log 2>&1
SALF_LIB=build_ab/nopf/libsalf_b200.so python tools/ab_raster.py init nopf >> gpurun_out/ab31.log 2>&1
python tools/ab_raster.py init pf2 >> gpurun_out/ab31.log 2>&1
