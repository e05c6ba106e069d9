# round-2 GPU call 46: host-side fixes (merged token ids from memoised per-chunk arrays, chunk text keys):
# full GPU suite, smoke, default-rule timeline, C3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r46_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r46_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r46_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r46_rc.txt
timeout 300 python scripts/dbg_timeline.py c3 0.2 5 > gpurun_out/r46_timeline.log 2>&1
timeout 900 python bench.py > gpurun_out/r46_bench_c3.json 2> gpurun_out/r46_bench_c3.err
echo "c3 rc=$?" >> gpurun_out/r46_rc.txt
echo done
