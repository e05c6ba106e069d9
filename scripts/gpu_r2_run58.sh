# round-2 GPU call 58: 3xTF32 pairs + 8-K-block phases: GPU suite, smoke, GEMM bench, full bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r58_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r58_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r58_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r58_smoke.log
timeout 300 python scripts/bench_gemm.py --only tf32x3 > gpurun_out/r58_gemm.log 2>&1
timeout 900 python bench.py > gpurun_out/r58_bench.json 2> gpurun_out/r58_bench.err
echo "bench rc=$?" >> gpurun_out/r58_bench.err
tail -n 3 gpurun_out/r58_gpu_tests.log; tail -n 2 gpurun_out/r58_smoke.log; cat gpurun_out/r58_gemm.log; head -c 400 gpurun_out/r58_bench.json; tail -n 2 gpurun_out/r58_bench.err
