"""Sum ncu --metrics gpu__time_duration.sum launch lists per kernel: python tools/launch_summary.py CSV"""
import collections, csv, sys
rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = list(csv.reader(rows)); h = r[0]; tot = collections.defaultdict(float); cnt = collections.Counter()
for x in r[1:]:
    d = dict(zip(h, x))
    if d.get("Metric Name") == "gpu__time_duration.sum":
        k = d["Kernel Name"][:70]; tot[k] += float(d["Metric Value"]); cnt[k] += 1
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    print(f"{v/1e3:10.1f} us total {cnt[k]:5d} launches {v/1e3/cnt[k]:9.1f} us avg  {k}")
