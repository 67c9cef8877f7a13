for k in 6 7 8 6 7 8; do SALF_OCT_JUMP=$k python tools/ab_ray.py jump$k >> gpurun_out/ab42.log 2>&1; done
