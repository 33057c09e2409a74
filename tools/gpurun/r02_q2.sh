# k_quant2 first GPU pass: suite (with the new scale tests) + bench
mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r02b/gpu_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b/bench_n1.json 2> gpurun_out/r02b/bench_n1.err; echo "bench rc=$?"
tail -3 gpurun_out/r02b/bench_n1.err; python -c "
import json;d=json.loads(open('gpurun_out/r02b/bench_n1.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['roofline'],d['kernels'])"
