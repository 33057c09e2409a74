# k_quant2: suite (empty-segment fix) + ncu of one RS-hop launch at the bench config
mkdir -p gpurun_out/r02c
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/r02c/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02c/gpu_tests.txt
timeout 300 python bench.py --profile-only > gpurun_out/r02c/plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 5 -c 1 -o gpurun_out/r02c/q2 python bench.py --profile-only > gpurun_out/r02c/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02c/ncu.log
