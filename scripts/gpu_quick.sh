# quick GPU loop: selected tests then a short bench (run under gpurun)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q ${TESTS:-} 2>&1 | tail -25 > gpurun_out/quick_tests.log
cat gpurun_out/quick_tests.log
if [ -z "${NOBENCH:-}" ]; then
timeout 600 python bench.py --skip-full --skip-e2e --skip-cpu ${BENCHARGS:-} > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'P'
import json
l=json.load(open("gpurun_out/quick_bench.json"))
print("TTFT", l["ms_per_step"], "clocks", l["clocks"])
for k,v in l["kernels"].items(): print(f"  {k:24s} {v}")
P
tail -3 gpurun_out/quick_bench.err
fi
