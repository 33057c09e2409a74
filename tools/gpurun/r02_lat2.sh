mkdir -p gpurun_out/r02lat
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_quant" -s 30 -c 1 -o gpurun_out/r02lat/tiny python tools/quant_latency.py > gpurun_out/r02lat/ncu_tiny.log 2>&1; echo "ncu rc=$?"
