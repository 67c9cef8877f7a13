python -m pytest tests -m gpu -x -q -k "march or ray or lidar or c3 or c4 or actor or octree or effects" > gpurun_out/t22.log 2>&1; echo rc=$? >> gpurun_out/t22.log
python tools/ab_ray.py mc6 > gpurun_out/ab13.log 2>&1
for v in 0 5 7 8; do SALF_LIB=build_ab/mc$v/libsalf_b200.so python tools/ab_ray.py mc$v >> gpurun_out/ab13.log 2>&1; done
