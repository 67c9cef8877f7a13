timeout 600 ./tools/div_check_bin > gpurun_out/divcheck.log 2>&1; echo rc=$? >> gpurun_out/divcheck.log
python -m pytest tests -m gpu -x -q -k "octree or march or query or lidar or ray or fisheye or c4 or actors" > gpurun_out/t53.log 2>&1; echo rc=$? >> gpurun_out/t53.log
for v in ddiv mark ddiv mark; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_ray.py $v >> gpurun_out/ab45.log 2>&1; done
