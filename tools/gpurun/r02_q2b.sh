# k_quant2 v2 (deferred arrivals, hoisted table loads, L2 prefetch): scale tests with per-test timeouts, suite, bench
mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_scale.py -v -x --timeout 300 -o faulthandler_timeout=280 --durations=0 > gpurun_out/r02d/scale.txt 2>&1; echo "scale rc=$?"
tail -40 gpurun_out/r02d/scale.txt
timeout 600 python -m pytest tests -m gpu -x -q --timeout 120 --deselect tests/test_gpu_scale.py > gpurun_out/r02d/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r02d/gpu_tests.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02d/bench_n1.json 2> gpurun_out/r02d/bench_n1.err; echo "bench rc=$?"
tail -3 gpurun_out/r02d/bench_n1.err; python -c "
import json;d=json.loads(open('gpurun_out/r02d/bench_n1.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['roofline'],d['kernels'])"
