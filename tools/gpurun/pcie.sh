mkdir -p gpurun_out/e2e
python tools/pcie_probe.py 2>&1 | tee gpurun_out/e2e/pcie.txt
nvidia-smi topo -m 2>&1 | head -12
