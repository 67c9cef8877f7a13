# ncu evidence for profiles/: one --set full capture of the top kernels of
# the C2 raster fwd+bwd and the C3 LiDAR (tools/ncu_target.py), and the
# launch list of one short bench run (cold-cache, serialised per-launch times).
ncu --set full --clock-control none --import-source on -k regex:"k_composite_fast|k_composite_redo|k_backward_fast|k_ray_forward_fast|k_ray_backward" -s 5 -c 5 -o gpurun_out/prof_full python tools/ncu_target.py > gpurun_out/ncu_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-profile > gpurun_out/ncu_launch_bench.log 2>&1
echo done
