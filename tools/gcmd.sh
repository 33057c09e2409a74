mkdir -p gpurun_out/r01b
timeout 600 python bench.py > gpurun_out/r01b/bench_n1.json.log 2> gpurun_out/r01b/bench_n1.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01b/bench_ref_n1.json.log 2>&1; echo ref rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01b/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_quant --launch-skip 21 --launch-count 1 -o gpurun_out/r01b/kq -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01b/ncu_kq.log 2>&1; echo kq rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply --launch-skip 20 --launch-count 1 -o gpurun_out/r01b/ka -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01b/ncu_ka.log 2>&1; echo ka rc=$?
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r01b/smi.txt
