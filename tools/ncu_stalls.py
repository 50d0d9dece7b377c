"""Summarise an `ncu --set full` raw CSV (ncu -i x.ncu-rep --page raw --csv): per kernel the time, DRAM bytes,
pipe utilisation and the warp-stall breakdown (stalled warps per issue slot)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}
base = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
for d in data:
    print(d[col["Kernel Name"]][:90])
    for b in base:
        if b in col:
            print(f"    {b:70s} {d[col[b]]:>14s} {units[col[b]]}")
    st = sorted(((float(d[col[h]].replace(',', '')), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                 for h in stalls), reverse=True)
    print("    stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:7]))
