compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_target.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck.log
compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python tools/sanitize_target.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck.log
compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_target.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/san_synccheck.log
