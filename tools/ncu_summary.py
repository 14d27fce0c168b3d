"""Summarise an ncu --set full report (raw page) into markdown for profiles/."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(raw))
h, units, v = rows[0], rows[1], rows[2]
get = {n: (x, u) for n, u, x in zip(h, units, v)}
keys = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("sm__warps_active.avg.per_cycle_active", "active warps/SM"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % (active)"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 traffic"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
print(f"# ncu summary: `{rep}`\n")
print("| metric | value |\n|---|---|")
for k, label in keys:
    if k in get:
        x, u = get[k]
        print(f"| {label} (`{k}`) | {x} {u} |")
stalls = [(n, float(get[n][0] or 0)) for n in get
          if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
stalls.sort(key=lambda t: -t[1])
print("\n| stall reason (warps per issue) | value |\n|---|---|")
for n, x in stalls[:10]:
    print(f"| {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} | {x:.3f} |")
