"""Top SASS stall sites of an ncu report: python tools/ncu_src_top.py REP [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src))); h = r[1]; d = r[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source"); iE = h.index("Instructions Executed")
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(x[iS] or 0) for x in d)
print("total samples", tot, "instructions", sum(float(x[iE] or 0) for x in d))
for idx, x in sorted(enumerate(d), key=lambda t: -float(t[1][iS] or 0))[:n]:
    why = sorted(((float(x[h.index(c)] or 0), c[6:]) for c in stalls), reverse=True)[:2]
    print(f"{idx:5d} {float(x[iS] or 0):7.0f} {x[iSrc][:60]:60s} {why}")
