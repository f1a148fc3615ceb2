"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel:
launches, total ms, share.  Usage: summarize_launches.py launches.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum": continue
    v = float(r[vi].replace(",", ""))
    v = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] in ("us", "usecond") else v)
    name = r[ki].split("(")[0][:90]
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"total {T:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{cnt[k]:6d} {v:9.3f} {100 * v / T:5.1f}%  {k}")
