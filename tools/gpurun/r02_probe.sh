# round 2, first call: TMEM-scratch probe + baseline suite + bench on this round's box
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/gpu.txt 2>&1
(cd tools/tmem_probe && timeout 120 ./probe) > gpurun_out/r02a/probe.txt 2>&1; echo "probe rc=$?"
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/gpu_tests.txt 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a/bench_n1.json 2> gpurun_out/r02a/bench_n1.err; echo "bench rc=$?"
nproc > gpurun_out/r02a/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/r02a/host.txt; free -g >> gpurun_out/r02a/host.txt
cat gpurun_out/r02a/probe.txt; tail -3 gpurun_out/r02a/gpu_tests.txt
