# round-2 GPU call 50: weight-streaming GEMV for M <= 4 bf16 GEMMs: kernel tests, decode A/B, API/parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemm or gemv" -s > gpurun_out/r50_tests.log 2>&1
echo "kernel tests rc=$?" >> gpurun_out/r50_rc.txt
for rep in 1 2; do
  CC_GEMM_GEMV=0 timeout 300 python scripts/bench_decode.py > gpurun_out/r50_decode_off_$rep.log 2>&1
  timeout 300 python scripts/bench_decode.py > gpurun_out/r50_decode_on_$rep.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r50_all.log 2>&1
echo "all rc=$?" >> gpurun_out/r50_rc.txt
echo done
