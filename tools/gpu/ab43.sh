python -m pytest tests/test_gpu_octree_jump.py -x -q > gpurun_out/t52.log 2>&1; echo rc=$? >> gpurun_out/t52.log
for v in lin brick lin brick; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_ray.py $v >> gpurun_out/ab44.log 2>&1; done
