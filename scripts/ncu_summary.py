"""Print the key metrics of an ncu report (details page)."""
import csv, subprocess, sys
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Eligible Warps Per Scheduler", "Issued Warp Per Scheduler",
        "Warp Cycles Per Issued Instruction", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy", "Block Limit Registers", "Achieved Active Warps Per SM"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]; ni = h.index("Metric Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit"); ki = h.index("Kernel Name")
    print("==", rep, r[1][ki][:70])
    seen = set()
    for x in r[1:]:
        if x[ni] in keys and x[ni] not in seen:
            seen.add(x[ni]); print(f"  {x[ni]:40s} {x[vi]} {x[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        i = rr[0].index(name); print(f"  {name:40s} {rr[2][i]} {rr[1][i]}")
