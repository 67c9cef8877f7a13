python -m pytest tests -m gpu -x -q > gpurun_out/t55.log 2>&1; echo rc=$? >> gpurun_out/t55.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench11.log 2>&1
