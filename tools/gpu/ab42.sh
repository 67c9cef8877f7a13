for v in nopf pf nopf pf; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_ray.py $v >> gpurun_out/ab43.log 2>&1; done
