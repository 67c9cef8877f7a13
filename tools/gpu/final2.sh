python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo rc=$? >> gpurun_out/smoke2.log
start=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/bench_default.log
