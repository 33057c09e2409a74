mkdir -p gpurun_out/r02s
timeout 300 python tools/nvlink_probe.py > gpurun_out/r02s/nvlink_probe.txt 2>&1; echo "probe rc=$?"
grep -E "delta [1-9]|links" gpurun_out/r02s/nvlink_probe.txt | head -20
timeout 1500 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02s/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|Error|passed|failed" gpurun_out/r02s/mg_tests.txt | head -20
