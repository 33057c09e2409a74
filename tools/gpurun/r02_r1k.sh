mkdir -p gpurun_out/r02q
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02q/bench.json 2> gpurun_out/r02q/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/r02q/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r02q/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()}, d['parity'])"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/r02q/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02q/gpu_tests.txt
