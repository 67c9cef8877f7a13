for v in rm4 rm5 rm6 rm8 cm4 cm8 rm4 rm6; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_ray.py $v >> gpurun_out/ab47.log 2>&1; done
