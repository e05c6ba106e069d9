# round-2 GPU call 65: scoring-cache prefix dedup on PCIe (CC_PREFIX_DEDUP): tests + e2e A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precompute.py tests/test_gpu_api.py -q -x -p no:cacheprovider > gpurun_out/r65_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r65_ab.log
for rep in 1 2; do
for d in 1 0; do
  CC_PREFIX_DEDUP=$d timeout 600 python bench.py --skip-full --skip-cpu > gpurun_out/r65_tmp.json 2> gpurun_out/r65_tmp.err
  python - $d <<'P' >> gpurun_out/r65_ab.log
import json,sys
l=json.load(open("gpurun_out/r65_tmp.json"))
sw=l["sweep"]
print("dedup", sys.argv[1], "ttft", round(l["ms_per_step"],2), "e2e", round(l["e2e"]["ms_per_step"],2), "h2d", l["e2e"]["h2d_bytes_per_step"], "clk", l["clocks"]["sm_mhz"], "e2e@5%", round(sw["0.05"]["e2e_ms"],2), "ttft@5%", round(sw["0.05"]["ttft_ms"],2), "e2e@10%", round(sw["0.10"]["e2e_ms"],2))
P
done
done
cat gpurun_out/r65_ab.log; tail -n 3 gpurun_out/r65_tests.log
