mkdir -p gpurun_out/final4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final4/build.log 2>&1 || { tail -20 gpurun_out/final4/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/final4/bench_n1.json 2> gpurun_out/final4/bench_n1.err; echo "n1 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final4/ref_n1.json 2> gpurun_out/final4/ref_n1.err; echo "ref rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2959$N bench.py --gpus $N > gpurun_out/final4/bench_n$N.json 2> gpurun_out/final4/bench_n$N.err; echo "n$N rc=$?"
done
for f in gpurun_out/final4/*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d.get('ms_per_step'),d.get('value'),(d.get('e2e') or {}).get('value'),(d.get('roofline') or {}).get('frac'), d.get('clocks'))"; done
