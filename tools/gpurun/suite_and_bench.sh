# GPU suite on the visible GPUs + N=1 bench (10 steps) + N=2 bench
mkdir -p gpurun_out/sb
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sb/build.log 2>&1 || { tail -20 gpurun_out/sb/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sb/n1_$i.json 2> gpurun_out/sb/n1.err
python -c "import json;d=json.loads(open('gpurun_out/sb/n1_$i.json').read().strip().splitlines()[-1]);k=d['kernels'];print('n1', round(d['ms_per_step'],3), round(sum(v['ms_per_step'] for n,v in k.items() if n.startswith('quant')),3), d['roofline']['frac'])"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sb/n2.json 2> gpurun_out/sb/n2.err
python -c "import json;d=json.loads(open('gpurun_out/sb/n2.json').read().strip().splitlines()[-1]);print('n2', round(d['ms_per_step'],3), d['value'])"
