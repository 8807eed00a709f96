"""Summarise an ncu --metrics gpu__time_duration.sum CSV: total time per kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows[start + 1:]:
    if len(r) > mv:
        name = r[kn].split("(")[0].replace("void ", "")
        tot[name] += float(r[mv].replace(",", "")) / 1e3; cnt[name] += 1
allt = sum(tot.values())
print(f"total {allt:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:12.1f} us {100*v/allt:5.1f}%  x{cnt[k]:5d}  {k}")
