timeout 900 ./tools/div_check_bin > gpurun_out/divcheck.log 2>&1; echo rc=$? >> gpurun_out/divcheck.log
