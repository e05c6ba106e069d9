# round-2 GPU call 34: norm_finalize with 32 loads in flight; C2 bench; C4
# (14B, 200K context) sequence-sharded at W=1 with the full-prefill denominator
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r34_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r34_rc.txt
timeout 600 python bench.py --config c2 --skip-cpu > gpurun_out/r34_bench_c2.json 2> gpurun_out/r34_bench_c2.err
echo "c2 rc=$?" >> gpurun_out/r34_rc.txt
timeout 1500 python bench.py --config c4 --sharded --steps 2 --warmup 1 > gpurun_out/r34_bench_c4.json 2> gpurun_out/r34_bench_c4.err
echo "c4 rc=$?" >> gpurun_out/r34_rc.txt
echo done
