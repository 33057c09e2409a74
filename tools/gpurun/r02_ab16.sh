# 1 GPU: k_apply occupancy (min blocks 4 / 5 per SM)
mkdir -p gpurun_out/r02ab16
for v in cur mb4 mb5 cur mb4 mb5; do
  env EMESH_LIB=build_var/lib$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02ab16/bench_$v.json 2> gpurun_out/r02ab16/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02ab16/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['avg_launch_ms'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'], d['parity']['cb_mismatches'])"
done
