mkdir -p gpurun_out/r02p
for S in 16 64 256; do
timeout 600 python bench.py --steps 5 --warmup 3 --S $S --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02p/bench_S$S.json 2> gpurun_out/r02p/bench_S$S.err; echo "bench S=$S rc=$?"
python -c "
import json;d=json.loads(open('gpurun_out/r02p/bench_S$S.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
