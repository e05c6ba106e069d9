# round-2 GPU call 36: PV parts 1/2/4 and the poly share under 4 parts, attention alone (C3 shape + dense 32K)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for lib in paper_2510_10129_b200/variants/libcc_pv1.so paper_2510_10129_b200/variants/libcc_pv2.so paper_2510_10129_b200/libcacheclip_sm100.so paper_2510_10129_b200/variants/libcc_poly3.so paper_2510_10129_b200/variants/libcc_poly5.so paper_2510_10129_b200/variants/libcc_poly6.so; do
  timeout 120 python scripts/bench_attention.py --lib $lib --dense 32768 >> gpurun_out/r36_attn.log 2>&1
done
done
timeout 120 python scripts/dbg_fa_trace.py paper_2510_10129_b200/variants/libcc_trace.so > gpurun_out/r36_trace4.log 2>&1
echo done
