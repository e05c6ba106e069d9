# round-2 GPU call 64: banked scoring attention with K/V prefetched two tiles ahead (two register sets):
# bitwise A/B of the scores, kernel/parity tests, timing A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=paper_2510_10129_b200/variants
for w in c2 c3; do
  timeout 300 python scripts/bt_bitwise.py gpurun_out/r64_new_$w.npy $w > gpurun_out/r64_bw.log 2>&1
  CACHECLIP_SM100_LIB=$V/libcc_bt0.so timeout 300 python scripts/bt_bitwise.py gpurun_out/r64_old_$w.npy $w >> gpurun_out/r64_bw.log 2>&1
  python -c "import numpy as np,sys; a=np.load('gpurun_out/r64_new_$w.npy'); b=np.load('gpurun_out/r64_old_$w.npy'); print('$w bitwise', a.shape==b.shape and bool((a.view(np.uint32)==b.view(np.uint32)).all()), float(np.abs(a-b).max()))" >> gpurun_out/r64_ab.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "banked or scale or parity or selection" > gpurun_out/r64_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r64_ab.log
for rep in 1 2; do
for lib in paper_2510_10129_b200/libcacheclip_sm100.so $V/libcc_bt0.so; do
  CACHECLIP_SM100_LIB=$lib timeout 400 python bench.py --skip-full --skip-e2e --skip-cpu --no-sweep > gpurun_out/r64_tmp.json 2> gpurun_out/r64_tmp.err
  python - $lib <<'P' >> gpurun_out/r64_ab.log
import json,sys
l=json.load(open("gpurun_out/r64_tmp.json"))
k=l["kernels"]
print(sys.argv[1].split('/')[-1], "ttft", round(l["ms_per_step"],2), "dr", round(l["default_rule"]["ttft_ms"],2), "clk", l["clocks"]["sm_mhz"], "banked", round(k["banked_attention_f32"]["ms_per_step"],3), "tf32", round(k["gemm_3xtf32"]["ms_per_step"],2))
P
done
done
rm -f gpurun_out/*.npy
cat gpurun_out/r64_ab.log; tail -n 3 gpurun_out/r64_tests.log
