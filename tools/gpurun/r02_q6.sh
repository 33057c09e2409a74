mkdir -p gpurun_out/r02m
for v in relax relaxnb; do
  L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02m/bench_$v.json 2> gpurun_out/r02m/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02m/bench_$v.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
