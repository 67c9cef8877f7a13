timeout 600 python -m pytest tests -m gpu -x -q -k "lidar or ray or octree" > gpurun_out/t58.log 2>&1; echo rc=$? >> gpurun_out/t58.log
for v in base kfeat base kfeat; do SALF_LIB=build_ab/$v/libsalf_b200.so timeout 300 python tools/ab_ray.py $v >> gpurun_out/ab51.log 2>&1; done
