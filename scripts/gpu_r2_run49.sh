# round-2 GPU call 49: decode per-launch times of one layer
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/bench_decode.py > gpurun_out/r49_decode.log 2>&1
echo done
