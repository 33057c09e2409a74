# 1 GPU: BIN lag (grids) x L2 policies (inputs evict-first, scratch evict-last)
mkdir -p gpurun_out/r02ab9
for v in cur el5 el8 lag8 el3 cur el5 el8; do
  env EMESH_LIB=build_var/lib$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02ab9/bench_$v.json 2> gpurun_out/r02ab9/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02ab9/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3),d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'])"
done
for v in cur el5 el3; do
  env EMESH_LIB=build_var/lib$v.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_quant" -c 16 --csv --log-file gpurun_out/r02ab9/ncu_$v.csv python bench.py --profile-only > /dev/null 2>&1; echo "ncu $v rc=$?"
  python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/r02ab9/ncu_$v.csv')))
for i,r in enumerate(rows):
    if 'Metric Name' in r: h=r; st=i; break
iK=h.index('Kernel Name'); iM=h.index('Metric Name'); iV=h.index('Metric Value'); iID=h.index('ID')
m={}
for r in rows[st+1:]:
    if len(r)!=len(h): continue
    m.setdefault(int(r[iID]),{'k':r[iK]})[r[iM]]=float(r[iV].replace(',',''))
for i,d in sorted(m.items()):
    if '<3>' in d['k']:
        print('$v', {k:d[k] for k in d if k!='k'}); break
PY
done
