python -m pytest tests -m gpu -x -q -k "deterministic or backward" > gpurun_out/t27.log 2>&1; echo rc=$? >> gpurun_out/t27.log
python tools/ab_raster.py init cur > gpurun_out/ab19.log 2>&1
