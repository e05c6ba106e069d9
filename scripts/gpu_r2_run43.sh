# round-2 GPU call 43: attention exp2 split placement (poly pairs spread / first / last), share, P parts
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_2510_10129_b200/variants
for rep in 1 2 3; do
for lib in paper_2510_10129_b200/libcacheclip_sm100.so $V/libcc_pos1.so $V/libcc_pos2.so $V/libcc_pv2.so $V/libcc_p5.so $V/libcc_p4.so $V/libcc_pos1p4.so $V/libcc_pos2p4.so; do
  timeout 120 python scripts/bench_attention.py --lib $lib --dense 32768 >> gpurun_out/r43_attn.log 2>&1
done
done
echo done
