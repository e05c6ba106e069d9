# round-2 GPU call 48: decode step composition under the launch profiler
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/bench_decode.py > gpurun_out/r48_decode.log 2>&1
CC_PDL=0 timeout 300 python scripts/bench_decode.py > gpurun_out/r48_decode_nopdl.log 2>&1
echo done
