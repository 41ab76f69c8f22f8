"""Summarise an ncu report: key metrics + SASS opcode/stall histogram."""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Executed Instructions",
        "Eligible Warps Per Scheduler", "No Eligible", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Block Limit Registers", "Block Limit Shared Mem", "Warp Cycles Per Issued Instruction", "Mem Pipes Busy")
rows = list(csv.reader(io.StringIO(det)))
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in keep:
        print(f"{d['Metric Name']:40s} {d['Metric Unit']:12s} {d['Metric Value']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    hh = rr[0]; vals = rr[2]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
                 "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                 "gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
        for i, n in enumerate(hh):
            if n == name:
                print(f"{name:60s} {rr[1][i]:10s} {vals[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
sr = list(csv.reader(io.StringIO(src)))
hdr = sr[1]; data = sr[2:]
if "Warp Stall Sampling (All Samples)" not in hdr:
    sys.exit(0)
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed")
ts = sum(float(r[iS] or 0) for r in data); ti = sum(float(r[iI] or 0) for r in data)
byop = collections.Counter(); bys = collections.Counter()
for r in data:
    t = r[1].strip().split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    byop[op] += float(r[iI] or 0); bys[op] += float(r[iS] or 0)
print("opcode     inst%  stall%")
for op, c in byop.most_common(22):
    print(f"{op:10s} {c/ti*100:5.1f}  {bys[op]/ts*100:5.1f}")
print("hottest stall sites:")
top = sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for i in sorted(top):
    print(f"{i:5d} {float(data[i][iS])/ts*100:5.1f}%  {data[i][1].strip()[:80]}")
