mkdir -p gpurun_out/r02o
timeout 300 python bench.py --profile-only > gpurun_out/r02o/plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 5 -c 1 -o gpurun_out/r02o/q2 python bench.py --profile-only > gpurun_out/r02o/ncu.log 2>&1; echo "ncu rc=$?"
tail -2 gpurun_out/r02o/ncu.log
