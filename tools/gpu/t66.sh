timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t66.log 2>&1; echo rc=$? >> gpurun_out/t66.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench14.log 2>&1
