# round-2 GPU call 57: scoring precision vs fp64 for 3xTF32 phase length / CTA pairs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_2510_10129_b200/variants
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 900 python scripts/diag_scoring_precision.py c2 c3 > gpurun_out/r57_$tag.log 2>&1
  for w in c2 c3; do cp gpurun_out/diag_scoring_$w.json gpurun_out/r57_${tag}_$w.json; done
}
run ph4_single CC_TF32_PAIR=0
run ph4_pair CC_TF32_PAIR=1
run ph8_pair CC_TF32_PAIR=1 CACHECLIP_SM100_LIB=$V/libcc_ph8.so
run ph8_single CC_TF32_PAIR=0 CACHECLIP_SM100_LIB=$V/libcc_ph8.so
tail -2 gpurun_out/r57_*.log
