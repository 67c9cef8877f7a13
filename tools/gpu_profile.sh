# Profile capture for profiles/ (run through gpurun, one GPU):
#  * ncu --set full of the hot kernels of tools/ncu_target.py (C2 raster forward + redo + backward,
#    C3 LiDAR forward + backward), second iteration (warm code, cold-ish data);
#  * the per-launch list of a short default bench run (gpu__time_duration, cold-cache, serialised).
# Then locally: python tools/ncu_summary.py gpurun_out/${TAG:-r2}_full.ncu-rep profiles/r2_ncu_full.md profiles/traffic.json
cd $GRAFT_REPO_ROOT
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_composite_fast|k_composite_redo|k_backward_hits|k_ray_forward_fast|k_ray_backward" -s 5 -c 5 \
  -o gpurun_out/${TAG:-r2}_full python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG:-r2}_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-profile \
  > gpurun_out/b_ncu.log 2>&1
