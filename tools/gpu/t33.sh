python -m pytest tests -m gpu -x -q -k "lidar or c3 or ray" > gpurun_out/t33.log 2>&1; echo rc=$? >> gpurun_out/t33.log
timeout 900 python bench.py --no-cpu > gpurun_out/bench7.log 2>&1
