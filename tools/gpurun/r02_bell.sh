mkdir -p gpurun_out/r02bell
timeout 900 python -m pytest tests/test_gpu_scale.py -q -s -k bell > gpurun_out/r02bell/out.txt 2>&1; echo "rc=$?"; tail -15 gpurun_out/r02bell/out.txt
