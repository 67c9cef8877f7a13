python -m pytest tests/test_gpu_octree_jump.py -x -q > gpurun_out/t50.log 2>&1; echo rc=$? >> gpurun_out/t50.log
for k in 0 4 5 6 3 0 4; do SALF_OCT_JUMP=$k python tools/ab_ray.py jump$k >> gpurun_out/ab41.log 2>&1; done
