for v in 4 6 8; do SALF_LIB=build_ab/ic$v/libsalf_b200.so python tools/ab_ray.py ic$v >> gpurun_out/ab15.log 2>&1; done
python tools/ab_ray.py nocache >> gpurun_out/ab15.log 2>&1
