# round-2 GPU call 51: GEMV L2 bulk prefetch of the weight rows before the dependency wait (0 / 4K / 16K / 64K per row)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_2510_10129_b200/variants
for rep in 1 2; do
for lib in $V/libcc_pf0.so $V/libcc_pf4k.so paper_2510_10129_b200/libcacheclip_sm100.so $V/libcc_pf64k.so; do
  timeout 300 python scripts/bench_decode.py --lib $lib > gpurun_out/r51_tmp.log 2>&1
  grep "ms/token" gpurun_out/r51_tmp.log >> gpurun_out/r51_decode.log
  grep "gemm_bf16 " gpurun_out/r51_tmp.log >> gpurun_out/r51_decode.log
done
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "gemv or qkv" > gpurun_out/r51_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r51_decode.log
echo done
