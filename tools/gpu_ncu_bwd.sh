# ncu --set full of the C2 raster backward + forward (tools/ncu_target.py), one launch each
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_backward|k_composite_fast" -s 2 -c 2 -o gpurun_out/r2_bwd_full python tools/ncu_target.py > gpurun_out/ncu_bwd.log 2>&1
