python tools/gpu/lid_time.py mb4 > gpurun_out/ab22.log 2>&1
for v in 6 8; do SALF_LIB=build_ab/rmb$v/libsalf_b200.so python tools/gpu/lid_time.py mb$v >> gpurun_out/ab22.log 2>&1; done
python tools/ab_ray.py mb4 >> gpurun_out/ab22.log 2>&1
for v in 6 8; do SALF_LIB=build_ab/rmb$v/libsalf_b200.so python tools/ab_ray.py mb$v >> gpurun_out/ab22.log 2>&1; done
