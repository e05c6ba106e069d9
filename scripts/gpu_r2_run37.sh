# round-2 GPU call 37: exp2 split (MUFU vs FMA-pipe polynomial share, degree 3/4) under 4 P parts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_2510_10129_b200/variants
for rep in 1 2; do
for lib in $V/libcc_pv1.so $V/libcc_poly4.so paper_2510_10129_b200/libcacheclip_sm100.so $V/libcc_poly2.so $V/libcc_deg3.so $V/libcc_deg3p4.so $V/libcc_deg3p5.so; do
  timeout 120 python scripts/bench_attention.py --lib $lib --dense 32768 >> gpurun_out/r37_attn.log 2>&1
done
done
echo done
