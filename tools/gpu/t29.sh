python -m pytest tests -m gpu -x -q -k "seed or train" > gpurun_out/t29.log 2>&1; echo rc=$? >> gpurun_out/t29.log
timeout 600 python bench.py --no-extras --no-cpu > gpurun_out/bench6.log 2>&1
