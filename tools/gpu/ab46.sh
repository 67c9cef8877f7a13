python -m pytest tests -m gpu -x -q -k "raster or certified or tile or stress or backward or deterministic" > gpurun_out/t54.log 2>&1; echo rc=$? >> gpurun_out/t54.log
for v in base assign base assign; do SALF_LIB=build_ab/$v/libsalf_b200.so python tools/ab_raster.py init $v >> gpurun_out/ab46.log 2>&1; done
