"""Summarise an .ncu-rep: key SOL / occupancy / stall metrics (run here, no GPU)."""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Executed Instructions", "Avg. Active Threads Per Warp",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Memory Throughput", "Dynamic Shared Memory Per Block", "Grid Size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    seen = set()
    for r in rows[1:]:
        name = r[mi]
        if name in KEYS and (r[ki], name) not in seen:
            seen.add((r[ki], name))
            print(f"{r[ki][:40]:40s} {name:40s} {r[vi]:>16s} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h = rr[0]
    want = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("_not_issued")]
    extra = [c for c in h if c in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                   "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
                                   "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
                                   "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active")]
    for row in rr[2:3]:
        vals = []
        for c in want:
            try:
                vals.append((float(row[h.index(c)].replace(",", "")), c))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1
        print("stall samples (top):")
        for v, c in sorted(vals, reverse=True)[:10]:
            print(f"   {c.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * v / tot:5.1f}%")
        for c in extra:
            print(f"   {c} = {row[h.index(c)]} {rr[1][h.index(c)]}")


if __name__ == "__main__":
    main(sys.argv[1])
