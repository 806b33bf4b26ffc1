"""Aggregate an ncu --metrics gpu__time_duration.sum launch list into per-kernel shares."""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")
    name = re.sub(r"^void\s+", "", name).replace("unnamed>::", "")
    v = float(d["Metric Value"])
    u = d["Metric Unit"]
    v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot/1e3:.2f} ms over {len(data)} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:32s} n={v[0]:5d} total={v[1]/1e3:9.2f}ms share={100*v[1]/tot:5.1f}% avg={v[1]/v[0]:9.1f}us")
