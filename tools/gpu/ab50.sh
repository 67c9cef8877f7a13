for v in blk128 blk32 blk64 blk256 blk128 blk64; do SALF_LIB=build_ab/$v/libsalf_b200.so timeout 300 python tools/ab_ray.py $v >> gpurun_out/ab50.log 2>&1; done
