# 1 GPU: STATS half-loop rolled (smaller kernel: fewer instruction-cache misses?) vs unrolled
mkdir -p gpurun_out/r02ab4
for v in new rolled new rolled; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02ab4/bench_$v.json 2> gpurun_out/r02ab4/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02ab4/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3),d['roofline']['avg_launch_ms'],d['roofline']['frac'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
