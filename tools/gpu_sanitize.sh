# compute-sanitizer memcheck / racecheck / synccheck on tools/sanitize_target.py (one GPU)
cd $GRAFT_REPO_ROOT
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
