cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_backward_fast|k_composite_fast" -s 2 -c 2 -o gpurun_out/r2_raster_full python tools/ncu_target.py > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_start.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --no-profile > gpurun_out/b_ncu.log 2>&1
ls -la gpurun_out
