# round-2 GPU call 55: phased 3xTF32 GEMMs on CTA pairs: kernel tests, full-size parity, GEMM A/B, bench A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "tf32" > gpurun_out/r55_kernels.log 2>&1
echo "kernel tests rc=$?" >> gpurun_out/r55_rc.txt
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/r55_parity.log 2>&1
echo "parity tests rc=$?" >> gpurun_out/r55_rc.txt
for p in 0 1; do
  echo "== CC_TF32_PAIR=$p" >> gpurun_out/r55_gemm.log
  CC_TF32_PAIR=$p timeout 300 python scripts/bench_gemm.py --only tf32x3 >> gpurun_out/r55_gemm.log 2>&1
done
for rep in 1 2; do
for p in 0 1; do
  CC_TF32_PAIR=$p timeout 400 python bench.py --skip-full --skip-e2e --skip-cpu --no-sweep > gpurun_out/r55_tmp.json 2> gpurun_out/r55_tmp.err
  python - $p <<'P' >> gpurun_out/r55_ab.log
import json,sys
l=json.load(open("gpurun_out/r55_tmp.json"))
k=l["kernels"]
print(sys.argv[1], "ttft", round(l["ms_per_step"],2), "dr", round(l["default_rule"]["ttft_ms"],2), "clk", l["clocks"]["sm_mhz"], "tf32", round(k["gemm_3xtf32"]["ms_per_step"],2), "n", k["gemm_3xtf32"]["launches_per_step"])
P
done
done
cat gpurun_out/r55_rc.txt; tail -3 gpurun_out/r55_kernels.log gpurun_out/r55_parity.log; cat gpurun_out/r55_gemm.log gpurun_out/r55_ab.log
