timeout 600 python -m pytest tests -m gpu -x -q -k "raster or certified or tile or stress or actors or c2" > gpurun_out/t56.log 2>&1; echo rc=$? >> gpurun_out/t56.log
for v in nobulk bulk nobulk bulk; do SALF_LIB=build_ab/$v/libsalf_b200.so timeout 300 python tools/ab_raster.py init $v >> gpurun_out/ab48.log 2>&1; done
SALF_LIB=build_ab/nobulk/libsalf_b200.so timeout 300 python tools/ab_raster.py surface nobulk_s >> gpurun_out/ab48.log 2>&1
SALF_LIB=build_ab/bulk/libsalf_b200.so timeout 300 python tools/ab_raster.py surface bulk_s >> gpurun_out/ab48.log 2>&1
