python -m pytest tests -m gpu -x -q > gpurun_out/t15.log 2>&1; echo rc=$? >> gpurun_out/t15.log
timeout 900 python bench.py --no-extras > gpurun_out/bench3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3.log
