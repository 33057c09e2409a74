# Round-2 final evidence on one GPU: GPU suite, smoke, bench (N=1) + reference arm, launch list, ncu --set full
mkdir -p gpurun_out/r02f1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f1/build.log 2>&1 || { tail -20 gpurun_out/r02f1/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r02f1/gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02f1/gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" > gpurun_out/r02f1/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02f1/smoke.txt
timeout 900 python bench.py > gpurun_out/r02f1/bench_n1.json 2> gpurun_out/r02f1/bench_n1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02f1/ref_n1.json 2> gpurun_out/r02f1/ref_n1.err; echo "ref rc=$?"
for f in bench_n1 ref_n1; do python -c "
import json;d=json.loads(open('gpurun_out/r02f1/$f.json').read().strip().splitlines()[-1]);print('$f',d.get('ms_per_step'),d.get('value'),(d.get('e2e') or {}).get('value'),(d.get('roofline') or {}).get('frac'),(d.get('cpu_baseline') or {}).get('value'), d.get('parity'), d.get('clocks'))"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f1/launches.csv python bench.py --steps 2 --warmup 1 --no-parity --no-e2e --no-cpu-baseline > gpurun_out/r02f1/launches.log 2>&1; echo "launches rc=$?"
timeout 300 python bench.py --profile-only > gpurun_out/r02f1/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_quant" -s 5 -c 1 -o gpurun_out/r02f1/kq python bench.py --profile-only > gpurun_out/r02f1/ncu_kq.log 2>&1; echo "ncu kq rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_apply" -s 2 -c 1 -o gpurun_out/r02f1/ka python bench.py --profile-only > gpurun_out/r02f1/ncu_ka.log 2>&1; echo "ncu ka rc=$?"
