mkdir -p gpurun_out/r02k
echo "== repro"; timeout 120 python tools/repro.py 2>&1 | tail -4
for v in default nopf w16; do
  L=""; [ $v != default ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02k/bench_$v.json 2> gpurun_out/r02k/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02k/bench_$v.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['roofline']['avg_launch_ms'],{k:v['ms_per_step'] for k,v in d['kernels'].items()})"
done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/r02k/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02k/gpu_tests.txt
