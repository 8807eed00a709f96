"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc, iall, inot = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Warp Stall Sampling (Not-issued Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr)]
tot = sum(float(r[iall] or 0) for r in body)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else None
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else None
print("total samples", tot)
if lo is not None:
    for r in body:
        a = int(r[ia], 16)
        if lo <= a <= hi:
            print(f"{r[ia]} {float(r[iall] or 0):7.0f} {float(r[inot] or 0):7.0f}  {r[isrc][:90]}")
else:
    for r in sorted(body, key=lambda r: -float(r[iall] or 0))[:n]:
        print(f"{r[ia]} {float(r[iall] or 0):7.0f} {float(r[inot] or 0):7.0f}  {r[isrc][:90]}")
