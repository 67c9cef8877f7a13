ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tile_order_block|k_tile_len_keys" -c 4 --csv python -c "
import sys, torch; sys.path.insert(0,'.')
from paper_2507_18713_b200 import configs, render_raster as RR
from paper_2507_18713_b200.scenes import get_scene
s=get_scene('S1M','init')
fb, st = RR.rasterize(s, configs.c2_camera(), return_state=True)
dc = torch.zeros((1080,1920,3), dtype=torch.float64, device='cuda')
for _ in range(2):
    st.tile_order = None
    RR.rasterize_backward(st, dc, None, as_dict=False)
" > gpurun_out/to_ncu.csv 2>&1
