python -m pytest tests -m gpu -x -q -k "raster or certified or actors" > gpurun_out/t13.log 2>&1; echo rc=$? >> gpurun_out/t13.log
python tools/ab_raster.py init np1 > gpurun_out/ab10.log 2>&1
for v in fnp2b4 fnp2b5 fnp2b6; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_raster.py init $v >> gpurun_out/ab10.log 2>&1; done
