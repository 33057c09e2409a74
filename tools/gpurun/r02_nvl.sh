# 2 GPUs: NVLink evidence (one process, two GPUs) + the NCCL slow-peer test
mkdir -p gpurun_out/r02u
timeout 600 python tools/nvlink_ncu.py > gpurun_out/r02u/nvlink_times.txt 2>&1; echo "nvlink_ncu rc=$?"; cat gpurun_out/r02u/nvlink_times.txt
timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"k_quant|k_apply" --csv --log-file gpurun_out/r02u/nvlink_ncu.csv \
  python tools/nvlink_ncu.py --iters 1 --warmup 0 > gpurun_out/r02u/nvlink_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 -k "slow_peer" > gpurun_out/r02u/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02u/mg_tests.txt | head
