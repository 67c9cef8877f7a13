for i in 1 2 3; do timeout 600 python bench.py --no-extras --no-cpu > gpurun_out/bench_e2e_$i.log 2>&1; done
