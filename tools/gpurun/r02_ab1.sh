# quantizer A/B on one GPU (config 2 bench, parity off), then the source-level ncu of k_quant<3>
mkdir -p gpurun_out/r02t
for v in base new rc newrc base new rc newrc; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02t/bench_$v.json 2> gpurun_out/r02t/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02t/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3),d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02t/gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02t/gpu_tests.txt
timeout 300 python bench.py --profile-only > gpurun_out/r02t/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 5 -c 1 -o gpurun_out/r02t/q1 python bench.py --profile-only > gpurun_out/r02t/ncu.log 2>&1; echo "ncu rc=$?"
