timeout 600 python -m pytest tests -m gpu -x -q -k "bin or raster or tile or c2" > gpurun_out/t57.log 2>&1; echo rc=$? >> gpurun_out/t57.log
for v in emit32 emit8 emit32 emit8; do SALF_LIB=build_ab/$v/libsalf_b200.so timeout 300 python tools/ab_raster.py init $v >> gpurun_out/ab49.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_emit -c 3 --csv python -c "
import sys; sys.path.insert(0,'.')
from paper_2507_18713_b200 import configs, render_raster as RR
from paper_2507_18713_b200.scenes import get_scene
s=get_scene('S1M','init')
for _ in range(3): RR.rasterize(s, configs.c2_camera())
" > gpurun_out/emit_ncu.csv 2>&1
