# round-2 GPU call 33: warp-wide elected tcgen05 issue (GEMMs, pair GEMM,
# attention), epilogue-specialised GEMM kernels: GPU suite, C3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r33_gpu.log 2>&1
echo "gpu rc=$?" >> gpurun_out/r33_rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r33_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r33_rc.txt
timeout 900 python bench.py > gpurun_out/r33_bench.json 2> gpurun_out/r33_bench.err
echo "bench rc=$?" >> gpurun_out/r33_rc.txt
echo done
