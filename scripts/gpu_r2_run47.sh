# round-2 GPU call 47: programmatic dependent launch for the per-layer kernels: full GPU suite, smoke,
# C3 A/B (CC_PDL=0 vs on), decode A/B, timeline
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r47_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r47_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r47_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r47_rc.txt
for rep in 1 2; do
  CC_PDL=0 timeout 600 python bench.py --skip-cpu --skip-full --no-sweep > gpurun_out/r47_c3_off_$rep.json 2>/dev/null
  timeout 600 python bench.py --skip-cpu --skip-full --no-sweep > gpurun_out/r47_c3_on_$rep.json 2>/dev/null
  CC_PDL=0 timeout 300 python scripts/bench_decode.py > gpurun_out/r47_decode_off_$rep.log 2>&1
  timeout 300 python scripts/bench_decode.py > gpurun_out/r47_decode_on_$rep.log 2>&1
done
timeout 300 python scripts/dbg_timeline.py c3 0.2 5 > gpurun_out/r47_timeline.log 2>&1
echo done
