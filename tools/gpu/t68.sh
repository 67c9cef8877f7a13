timeout 900 python -m pytest tests -m gpu -x -q -k "raster or certified or tile or stress or c2 or pins" > gpurun_out/t68.log 2>&1; echo rc=$? >> gpurun_out/t68.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_composite_redo -c 3 --csv python -c "
import sys; sys.path.insert(0,'.')
from paper_2507_18713_b200 import configs, render_raster as RR
from paper_2507_18713_b200.scenes import get_scene
s=get_scene('S1M','init')
for _ in range(3): RR.rasterize(s, configs.c2_camera())
" > gpurun_out/redo_ncu.csv 2>&1
