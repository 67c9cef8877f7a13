python tools/ab_ray.py base > gpurun_out/ab24.log 2>&1
for v in rb5 rb6; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_ray.py $v >> gpurun_out/ab24.log 2>&1; done
python tools/ab_raster.py init base >> gpurun_out/ab24.log 2>&1
SALF_LIB=build_ab/cf4/libsalf_b200.so python tools/ab_raster.py init cf4 >> gpurun_out/ab24.log 2>&1
