mkdir -p gpurun_out/e2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e/build.log 2>&1 || { tail -20 gpurun_out/e2e/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ring.py -q -x 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e/n1.json 2> gpurun_out/e2e/n1.err; echo "n1 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/e2e/n1.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['e2e'])"
