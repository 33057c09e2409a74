"""Summarise an ncu report: per kernel time, DRAM bytes, throughput, stalls."""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
def col(r, name):
    return r[h.index(name)] if name in h else ""
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
stalls = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print("==", col(r, "Kernel Name"), "grid", col(r, "launch__grid_size"))
    for w in want:
        if w in h: print(f"   {w:70s} {col(r, w)} {rows[1][h.index(w)]}")
    st = sorted(((float(col(r, c) or 0), c) for c in stalls), reverse=True)[:6]
    print("   top stalls:", ", ".join(f"{c.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, c in st))
