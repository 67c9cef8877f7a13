start=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/bench_default.log
start=$(date +%s); timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$? secs=$(( $(date +%s) - start ))" >> gpurun_out/bench_ref.log
