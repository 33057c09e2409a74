mkdir -p gpurun_out/r02t
for v in default rc default rc; do
  L=""; [ $v != default ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02t/bench_$v.json 2> gpurun_out/r02t/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02t/bench_$v.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
timeout 300 python bench.py --profile-only > gpurun_out/r02t/plain.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 5 -c 1 -o gpurun_out/r02t/q1 python bench.py --profile-only > gpurun_out/r02t/ncu.log 2>&1; echo "ncu rc=$?"
