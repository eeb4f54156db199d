"""Summarise an ncu report: time, DRAM traffic, FP64 pipe, occupancy, issue, top stall reasons per kernel."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("launch__registers_per_thread", "regs"), ("launch__occupancy_limit_registers", "occ_lim_regs"),
        ("launch__occupancy_limit_shared_mem", "occ_lim_smem"), ("lts__t_sector_hit_rate.pct", "L2hit%"),
        ("l1tex__t_sector_hit_rate.pct", "L1hit%"), ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
        ("sm__cycles_elapsed.avg.per_second", "clk")]
for d in data:
    print("=====", d[ix["Kernel Name"]], d[ix.get("Grid Size", 0)] if "Grid Size" in ix else "")
    for k, name in KEYS:
        if k in ix:
            print(f"  {name:14s} {d[ix[k]]:>16s} {units[ix[k]]}")
    items = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                items.append((float(d[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in items) or 1
    print("  stalls: " + ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in sorted(items, reverse=True)[:6]))
    fp = 0
    for op in ("dfma", "dadd", "dmul"):
        k = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
        if k in ix:
            fp += float(d[ix[k]])
    print(f"  fp64 thread-inst per cycle (chip): {fp:.0f} of 9472")
