"""Key metrics per launch from an `ncu --page raw --csv` export (dev tool)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
data = [r for r in rows[2:] if len(r) == len(hdr)]
want = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "ms"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64inst%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("launch__registers_per_thread", "regs"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "lanes/inst"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("smsp__inst_executed.sum", "warp_inst"), ("launch__grid_size", "grid")]
idx = {h: i for i, h in enumerate(hdr)}
units = rows[1]
for r in data:
    out = []
    for k, nm in want:
        if k in idx:
            v = r[idx[k]]
            u = units[idx[k]]
            out.append(f"{nm}={v[:60] if nm=='kernel' else v}{'' if nm=='kernel' else (' '+u if u else '')}")
    print(" | ".join(out))
