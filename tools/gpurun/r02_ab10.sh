# 1 GPU: virtual ring decodes each final payload once for all local replicas (new) vs once per replica (old)
mkdir -p gpurun_out/r02ab10
for v in old new3 old new3; do
  env EMESH_LIB=build_var/lib$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02ab10/bench_$v.json 2> gpurun_out/r02ab10/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02ab10/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['hbm_frac_step'], {k:(round(v['ms_per_step'],3), v['launches_per_step']) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'], d['parity']['theta_mismatches'], d['parity']['momentum_mismatches'])"
done
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r02ab10/tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02ab10/tests.txt
