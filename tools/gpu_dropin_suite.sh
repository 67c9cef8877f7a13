# the reference's hot-path tests on the drop-in backend, both precisions (summaries in gpurun_out/)
cd $GRAFT_REPO_ROOT/baseline/_ref/salf_tests
for p in fp64 mixed; do
SALF_DROPIN_PRECISION=$p SALF_DROPIN_REPORT=1 PYTHONPATH=$GRAFT_REPO_ROOT/baseline/_ref:$GRAFT_REPO_ROOT:$GRAFT_REPO_ROOT/tests timeout 900 python -m pytest -q -p _dropin_plugin -p no:cacheprovider -rf test_render_raster.py test_render_ray.py test_octree.py test_backward.py > $GRAFT_REPO_ROOT/gpurun_out/dropin_suite_$p.txt 2>&1
done
