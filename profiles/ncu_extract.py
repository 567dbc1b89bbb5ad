"""Key metrics of every kernel in an ncu --set full report (ncu -i ... --page raw --csv).

    python profiles/ncu_extract.py report.ncu-rep|raw.csv [--json out.json]

Prints duration, DRAM/L2 traffic, issue and pipe utilisations, the per-pipe warp-instruction counts
(sm__inst_executed_pipe_*.sum, the instruction mix the ALU roofline of bench.py uses) and the top
stall reasons."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "lts__t_bytes.sum.per_second", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
PIPES = ["alu", "fma", "fmaheavy", "fmalite", "fp64", "lsu", "adu", "cbu", "uniform", "xu"]


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def main():
    rep = sys.argv[1]
    if rep.endswith(".csv"):   # an exported raw page (ncu -i rep --page raw --csv > x.csv)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name"), "metrics": {}, "pipe_warp_inst": {}}
        print(d.get("Kernel Name"))
        for key in KEYS:
            if key in d:
                print(f"  {key} = {d.get(key)} {u.get(key, '')}")
                k["metrics"][key] = [num(d.get(key)), u.get(key, "")]
        for p in PIPES:
            key = f"sm__inst_executed_pipe_{p}.sum"
            if key in d and num(d[key]) is not None:
                k["pipe_warp_inst"][p] = num(d[key])
        print("  pipe warp-instructions:", k["pipe_warp_inst"])
        st = {key: num(v) for key, v in d.items() if key.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not key.endswith("not_issued") and num(v) is not None}
        tot = sum(st.values()) or 1
        k["stalls"] = [(key.replace("smsp__pcsamp_warps_issue_stalled_", ""), round(100 * v / tot, 1))
                       for key, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]]
        print("  stalls:", k["stalls"])
        res.append(k)
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
