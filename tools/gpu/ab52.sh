timeout 600 python -m pytest tests -m gpu -x -q -k "lidar or ray or octree" > gpurun_out/t59.log 2>&1; echo rc=$? >> gpurun_out/t59.log
for v in noearly early early_b5 noearly early early_b5; do SALF_LIB=build_ab/$v/libsalf_b200.so timeout 300 python tools/ab_ray.py $v >> gpurun_out/ab52.log 2>&1; done
