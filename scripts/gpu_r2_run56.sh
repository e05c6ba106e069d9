# round-2 GPU call 56: 3xTF32 phase length vs CTA pairs (timing only; phases 4 = default lib)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_2510_10129_b200/variants
for lib in paper_2510_10129_b200/libcacheclip_sm100.so $V/libcc_ph8.so $V/libcc_ph64.so; do
for p in 0 1; do
  echo "== $lib CC_TF32_PAIR=$p" >> gpurun_out/r56_gemm.log
  CC_TF32_PAIR=$p timeout 300 python scripts/bench_gemm.py --lib $lib --only tf32x3 >> gpurun_out/r56_gemm.log 2>&1
done
done
cat gpurun_out/r56_gemm.log
