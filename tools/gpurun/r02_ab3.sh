# quantizer A/B: table replication x smem carveout (L1 size)
mkdir -p gpurun_out/r02z
for v in base new rep1c64 rep4 rep16 base new rep1c64 rep4 rep16; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02z/bench_$v.json 2> gpurun_out/r02z/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02z/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3),d['roofline']['avg_launch_ms'],d['roofline']['frac'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,launch__shared_mem_config_size,sm__warps_active.avg.pct_of_peak_sustained_active
for v in base new rep16; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 ncu --metrics $M --clock-control none -k regex:k_quant -c 16 --csv --log-file gpurun_out/r02z/ncu_$v.csv python bench.py --profile-only > gpurun_out/r02z/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
