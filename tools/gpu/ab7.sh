python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
python tools/ab_raster.py init cur > gpurun_out/ab7.log 2>&1
SALF_LIB=build_ab/fwdb2/libsalf_b200.so python tools/ab_raster.py init fwdb2 >> gpurun_out/ab7.log 2>&1
for v in fm1 fm2 fm4; do SALF_NO_REDO=1 SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_raster.py init $v >> gpurun_out/ab7.log 2>&1; done
SALF_NO_REDO=1 python tools/ab_raster.py init noredo >> gpurun_out/ab7.log 2>&1
