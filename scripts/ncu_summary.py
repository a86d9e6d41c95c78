"""Summarise an ncu --set full report (one kernel) into text: SOL, DRAM traffic, pipes, stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(name):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


d = page("details")
h = d[0]
keep = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block", "Achieved Occupancy", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "SM Frequency"]
name = None
for row in d[1:]:
    r = dict(zip(h, row))
    name = r["Kernel Name"]
    if r["Metric Name"] in keep:
        print(f"{r['Section Name'][:34]:34s} {r['Metric Name']:38s} {r['Metric Value']} {r['Metric Unit']}")
raw = page("raw")
h, u, v = raw[0], raw[1], raw[2]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]
print("kernel:", name)
for i, n in enumerate(h):
    if n in want or n.startswith("sm__pipe_tcgen05") or n.startswith("sm__pipe_tma"):
        if v[i] not in ("", "0"):
            print(f"  {n} = {v[i]} {u[i]}")
st = [(n, v[i]) for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
tot = sum(float(x or 0) for _, x in st)
print("warp stall samples (share):")
for n, x in sorted(st, key=lambda p: -float(p[1] or 0))[:10]:
    print(f"  {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {float(x) / tot * 100:5.1f}%")
