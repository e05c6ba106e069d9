# round-2 GPU call 10: split-K bf16 GEMM for few-row launches: kernel tests,
# GPU suite, same-box A/B of the small-grid splits (attention split-KV and
# GEMM split-K) on the C3 sweep incl. the default rule, launch list, decode
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm or attention" > gpurun_out/r10_kernels.log 2>&1
echo "kernels rc=$?" >> gpurun_out/r10_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r10_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r10_rc.txt
B="--skip-cpu --skip-e2e --steps 5"
timeout 900 python bench.py $B > gpurun_out/r10_bench_a.json 2> gpurun_out/r10_bench_a.err
CC_ATTN_SPLIT=0 CC_GEMM_SPLITK=0 timeout 900 python bench.py $B > gpurun_out/r10_bench_off.json 2> gpurun_out/r10_bench_off.err
timeout 900 python bench.py $B > gpurun_out/r10_bench_b.json 2> gpurun_out/r10_bench_b.err
OUT=r10_launches_dr05 BENCHARGS="--ratio 0.05 --window-threshold 5 --no-sweep" sh scripts/launch_list.sh
timeout 600 python scripts/bench_decode.py > gpurun_out/r10_decode.log 2>&1
CC_GEMM_SPLITK=0 timeout 600 python scripts/bench_decode.py > gpurun_out/r10_decode_off.log 2>&1
echo done
