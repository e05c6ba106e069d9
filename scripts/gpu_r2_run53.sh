# round-2 GPU call 53: assembly grid cap (CC_ASSEMBLE_CTAS) A/B on C3 20% + default rule
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for n in 0 148 296 592 1184; do
  CC_ASSEMBLE_CTAS=$n timeout 400 python bench.py --skip-full --skip-e2e --skip-cpu --no-sweep > gpurun_out/r53_tmp.json 2> gpurun_out/r53_tmp.err
  python - $n <<'P' >> gpurun_out/r53_ab.log
import json,sys
l=json.load(open("gpurun_out/r53_tmp.json"))
k=l["kernels"]
print(sys.argv[1], "ttft", round(l["ms_per_step"],2), "dr", round(l["default_rule"]["ttft_ms"],2), "clk", l["clocks"]["sm_mhz"], "asm", round(k["assemble_kv"]["ms_per_step"],3), "tf32", round(k["gemm_3xtf32"]["ms_per_step"],2))
P
done
done
cat gpurun_out/r53_ab.log
