for v in old new; do
SALF_LIB=build_ab/$v/libsalf_b200.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_composite_redo -c 3 --csv python -c "
import sys; sys.path.insert(0,'.')
from paper_2507_18713_b200 import configs, render_raster as RR
from paper_2507_18713_b200.scenes import get_scene
s=get_scene('S1M','init')
for _ in range(3): RR.rasterize(s, configs.c2_camera())
" > gpurun_out/redo_ncu_$v.csv 2>&1
done
