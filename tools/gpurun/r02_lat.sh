mkdir -p gpurun_out/r02lat
timeout 300 python tools/quant_latency.py > gpurun_out/r02lat/lat.txt 2>&1; echo "rc=$?"; cat gpurun_out/r02lat/lat.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_quant" -c 60 --csv --log-file gpurun_out/r02lat/ncu.csv python tools/quant_latency.py > gpurun_out/r02lat/ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/r02lat/ncu.csv')))
for i,r in enumerate(rows):
    if 'Metric Name' in r: h=r; st=i; break
iG=h.index('Grid Size'); iV=h.index('Metric Value')
vals=[(r[iG], float(r[iV].replace(',',''))) for r in rows[st+1:] if len(r)==len(h)]
import collections
d=collections.defaultdict(list)
for g,v in vals: d[g].append(v)
for g,v in d.items(): print('grid', g, 'launches', len(v), 'median us', sorted(v)[len(v)//2]/1e3)
PY
