python -m pytest tests -m gpu -x -q -k "march or ray or lidar or c3 or c4 or actor or octree or effects or query or stress or raw" > gpurun_out/t38.log 2>&1; echo rc=$? >> gpurun_out/t38.log
python tools/ab_ray.py fastdiv > gpurun_out/ab29.log 2>&1
SALF_LIB=build_ab/nofd/libsalf_b200.so python tools/ab_ray.py nofd >> gpurun_out/ab29.log 2>&1
python tools/gpu/lid_time.py fastdiv >> gpurun_out/ab29.log 2>&1
SALF_LIB=build_ab/nofd/libsalf_b200.so python tools/gpu/lid_time.py nofd >> gpurun_out/ab29.log 2>&1
