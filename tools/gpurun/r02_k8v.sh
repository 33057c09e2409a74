# 1 GPU: k = 8 DiLoCo workers on one GPU (virtual ring) at 1B params/worker: the k = 8 plan, 7 hops, parity sample
mkdir -p gpurun_out/r02k8
timeout 900 python bench.py --workers 8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02k8/bench_k8.json 2> gpurun_out/r02k8/bench_k8.err; echo "k8 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02k8/bench_k8.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), d['value'], d['roofline']['frac'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity'])"
