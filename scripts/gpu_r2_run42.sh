# round-2 GPU call 42: banded schedule in the single-CTA GEMM too: full GPU suite, smoke, default C3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r42_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r42_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r42_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r42_rc.txt
timeout 900 python bench.py > gpurun_out/r42_bench_c3.json 2> gpurun_out/r42_bench_c3.err
echo "c3 rc=$?" >> gpurun_out/r42_rc.txt
echo done
