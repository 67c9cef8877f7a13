timeout 900 python -m pytest tests -m gpu -x -q -k "train or rig or lidar" > gpurun_out/t63.log 2>&1; echo rc=$? >> gpurun_out/t63.log
timeout 600 python tools/prof_c5_parts.py > gpurun_out/c5parts2.log 2>&1
