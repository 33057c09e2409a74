# Virtual ring: chunk c's decodes on s_comm overlapping chunk c+1's chain (EMESH_VIRTUAL_OVERLAP) — parity + A/B
mkdir -p gpurun_out/vov
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/vov/build.log 2>&1 || { tail -20 gpurun_out/vov/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_codec.py -x -q 2>&1 | tail -3
for rep in 1 2 3; do for v in 0 1; do
EMESH_VIRTUAL_OVERLAP=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vov/ov${v}_$rep.json 2> gpurun_out/vov/ov$v.err
python -c "import json;d=json.loads(open('gpurun_out/vov/ov${v}_$rep.json').read().strip().splitlines()[-1]);print('ov=$v', round(d['ms_per_step'],3), d['value'], d['clocks'])"
done; done
timeout 600 python bench.py > gpurun_out/vov/bench_n1.json 2> gpurun_out/vov/bench_n1.err; echo "bench rc=$?"; tail -c 600 gpurun_out/vov/bench_n1.json
