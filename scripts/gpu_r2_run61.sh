# round-2 GPU call 61: HEAD check (tf32 pair tests added) (GPU suite, smoke, default bench)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r61_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r61_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r61_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r61_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r61_smoke.log
timeout 900 python bench.py > gpurun_out/r61_bench.json 2> gpurun_out/r61_bench.err
echo "bench rc=$?" >> gpurun_out/r61_bench.err
tail -3 gpurun_out/r61_gpu_tests.log; tail -2 gpurun_out/r61_smoke.log; head -c 600 gpurun_out/r61_bench.json; tail -2 gpurun_out/r61_bench.err
