# round-2 GPU call 38: attention with 4 P parts + degree-3 polynomial share: full GPU suite, smoke, C3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r38_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r38_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r38_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r38_rc.txt
timeout 600 python bench.py > gpurun_out/r38_bench_c3.json 2> gpurun_out/r38_bench_c3.err
echo "c3 rc=$?" >> gpurun_out/r38_rc.txt
timeout 120 python scripts/bench_attention.py --dense 32768 >> gpurun_out/r38_attn.log 2>&1
echo done
