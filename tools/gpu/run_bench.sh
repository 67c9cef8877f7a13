python -m pytest tests/test_gpu_edge.py -m gpu -x -q -k "certified" > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
timeout 900 python bench.py > gpurun_out/bench2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2.log
