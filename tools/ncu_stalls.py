"""Sum warp-stall reasons over an address range of an ncu source CSV (sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
ia, isrc = hdr.index("Address"), hdr.index("Source")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 64
tot = {hdr[i]: 0.0 for i in cols}
n = 0
for r in body:
    a = int(r[ia], 16)
    if lo <= a <= hi:
        n += 1
        for i in cols:
            tot[hdr[i]] += float(r[i] or 0)
s = sum(tot.values())
print(f"{n} instructions, {s:.0f} samples")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v > 0: print(f"  {k:28s} {v:8.0f} {100*v/s:5.1f}%")
