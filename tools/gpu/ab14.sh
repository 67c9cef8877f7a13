python -m pytest tests -m gpu -x -q -k "march or ray or lidar or c3 or c4 or actor or octree or effects or query" > gpurun_out/t23.log 2>&1; echo rc=$? >> gpurun_out/t23.log
python tools/ab_ray.py intbits > gpurun_out/ab14.log 2>&1
SALF_LIB=build_ab/ib0/libsalf_b200.so python tools/ab_ray.py fma_update >> gpurun_out/ab14.log 2>&1
SALF_LIB=build_ab/orig/libsalf_b200.so python tools/ab_ray.py orig >> gpurun_out/ab14.log 2>&1
