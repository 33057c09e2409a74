# Configs 3 / 5 / 4 at 4 GPUs (and the k=2 sweep on GPUs 0-1) with the current build
mkdir -p gpurun_out/cfg
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cfg/build.log 2>&1 || exit 1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 4 --tensors intellect1 --S 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg/bench_n4_cfg5_S4.json 2> gpurun_out/cfg/cfg5.err; echo "cfg5 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --params 10211381248 --S 80 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg/bench_n4_10b_S80.json 2> gpurun_out/cfg/10b.err; echo "10b rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 tools/sweep_msg.py 4294967296 5 > gpurun_out/cfg/sweep_n4.jsonl 2> gpurun_out/cfg/sweep4.err; echo "sweep4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29634 tools/sweep_msg.py 1073741824 5 > gpurun_out/cfg/sweep_n2.jsonl 2> gpurun_out/cfg/sweep2.err; echo "sweep2 rc=$?"
for f in gpurun_out/cfg/bench_*.json; do python -c "
import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['ms_per_step'],2), d['value'])"; done
cat gpurun_out/cfg/sweep_n4.jsonl | tail -12
cat gpurun_out/cfg/sweep_n2.jsonl | tail -10
