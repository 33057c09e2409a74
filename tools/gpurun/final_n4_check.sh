# Final HEAD on 4 GPUs: GPU suite (4-GPU parity cases included) + N=4 and N=2 bench lines
mkdir -p gpurun_out/f4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f4/build.log 2>&1 || { tail -20 gpurun_out/f4/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 2969$N bench.py --gpus $N > gpurun_out/f4/bench_n$N.json 2> gpurun_out/f4/bench_n$N.err; echo "n$N rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/f4/bench_n$N.json').read().strip().splitlines()[-1]);print('n$N', round(d['ms_per_step'],3), d['value'], d['e2e']['value'], d['clocks'])"
done
