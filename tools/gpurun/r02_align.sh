mkdir -p gpurun_out/r02e
echo "== default"; CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/repro.py 2>&1 | tail -4
echo "== no prefetch"; CUDA_LAUNCH_BLOCKING=1 EMESH_LIB=build_var/libnopf.so timeout 120 python tools/repro.py 2>&1 | tail -4
