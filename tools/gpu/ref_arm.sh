python -m pytest tests -m gpu -x -q > gpurun_out/t21.log 2>&1; echo rc=$? >> gpurun_out/t21.log
( time timeout 900 python bench.py --impl reference --steps 2 --warmup 3 ) > gpurun_out/ref_arm.log 2>&1; echo "ref rc=$?" >> gpurun_out/ref_arm.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke2.log
