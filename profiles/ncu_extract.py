"""Key metrics of every kernel in an ncu --set full report (ncu -i ... --page raw --csv)."""
import csv, io, subprocess, sys
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r)); u = dict(zip(hdr, units))
    print(d.get("Kernel Name"))
    for k in KEYS:
        print(f"  {k} = {d.get(k)} {u.get(k, '')}")
    st = {k: float(v.replace(',', '')) for k, v in d.items() if k.startswith('smsp__pcsamp_warps_issue_stalled_')
          and not k.endswith('not_issued') and v.replace(',', '').replace('.', '').isdigit()}
    tot = sum(st.values()) or 1
    print("  stalls:", [(k.replace('smsp__pcsamp_warps_issue_stalled_', ''), round(100 * v / tot, 1))
                        for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:5]])
