"""Top SASS instructions by warp-stall samples (with stall breakdown) from an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kfilter = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kfilter:
    cmd += ["-k", kfilter]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
rd = csv.reader(io.StringIO("\n".join(lines[i:])))
hdr = next(rd)
rows = [r for r in rd if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
def num(x):
    try: return float(x)
    except ValueError: return 0.0
tot = sum(num(r[si]) for r in rows)
agg = {hdr[k]: sum(num(r[k]) for r in rows) for k in stall_cols}
print("total samples", tot)
print("kernel-wide:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
rows.sort(key=lambda r: -num(r[si]))
for r in rows[:top]:
    br = sorted(((hdr[k][6:], num(r[k])) for k in stall_cols), key=lambda kv: -kv[1])[:2]
    print(f"{int(num(r[si])):7d} {100*num(r[si])/tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} {br}")
