# round-2 GPU call 66: final HEAD check (GPU suite, smoke, default bench)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r66_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r66_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r66_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r66_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r66_smoke.log
timeout 900 python bench.py > gpurun_out/r66_bench.json 2> gpurun_out/r66_bench.err
echo "bench rc=$?" >> gpurun_out/r66_bench.err
tail -3 gpurun_out/r66_gpu_tests.log; tail -2 gpurun_out/r66_smoke.log; head -c 600 gpurun_out/r66_bench.json; tail -2 gpurun_out/r66_bench.err
