"""Turn a gpurun_out/prof capture (tools/capture_profiles.sh) into the tracked
summaries under profiles/:

  profiles/<tag>_bench.json         the bench line of the capture run (no profiler)
  profiles/<tag>_launches.txt       per-kernel share of the ncu launch list
  profiles/<tag>_ncu_<kernel>.txt   key --set full metrics + top stalled SASS lines
  profiles/ncu_traffic.json         dram read+write bytes per launch (read by bench.py)

usage: python tools/summarize_profiles.py <tag> [prof_dir]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "L2 Hit Rate", "Block Size", "Grid Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw_metrics(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", str(rep), "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for k in RAW:
        for i, h in enumerate(hdr):
            if h.endswith(k) or h == k:
                out[k] = (vals[i], units[i])
                break
    return out, hdr[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "", vals[hdr.index("Kernel Name")]


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    tag = sys.argv[1]
    prof = Path(sys.argv[2]) if len(sys.argv) > 2 else REPO / "gpurun_out" / "prof"
    dst = REPO / "profiles"
    dst.mkdir(exist_ok=True)
    if (prof / "bench.json").exists():
        (dst / f"{tag}_bench.json").write_text((prof / "bench.json").read_text())
    for name, cmd in (("launches", "python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary (FP64)"),
                      ("launches_fp32", "python bench.py --dtype fp32 --steps 1 --warmup 3 --no-cpu-baseline "
                                        "--no-secondary")):
        if (prof / f"{name}.csv").exists():
            out = subprocess.run([sys.executable, str(REPO / "tools" / "launches.py"), str(prof / f"{name}.csv")],
                                 capture_output=True, text=True).stdout
            (dst / f"{tag}_{name}.txt").write_text(
                "# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised launches) of\n"
                f"# {cmd}; per-kernel totals and share\n" + out)
    traffic_path = dst / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    for rep in sorted(prof.glob("full_*.ncu-rep")):
        kern = rep.stem[len("full_"):]
        det = list(csv.reader(io.StringIO(ncu("-i", str(rep), "--page", "details", "--csv"))))
        lines = [f"# ncu --set full --clock-control none, one launch of {kern} (tools/capture_profiles.sh)"]
        if det:
            hdr = det[0]
            name_i = hdr.index("Kernel Name")
            mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
            lines.append(f"kernel: {det[1][name_i]}")
            seen = set()
            for r in det[1:]:
                if len(r) > vi and r[mi] in KEYS and r[mi] not in seen:
                    seen.add(r[mi])
                    lines.append(f"{r[mi]:32s} {r[vi]} {r[ui]}")
        raw, _, _ = raw_metrics(rep)
        for k, (v, u) in raw.items():
            lines.append(f"{k:32s} {v} {u}")
        if "dram__bytes_read.sum" in raw and "dram__bytes_write.sum" in raw:
            tb = to_bytes(*raw["dram__bytes_read.sum"]) + to_bytes(*raw["dram__bytes_write.sum"])
            traffic[kern] = tb
            lines.append(f"{'traffic (read+write) bytes':32s} {tb:.4g}")
        hot = subprocess.run([sys.executable, str(REPO / "tools" / "ncu_hot.py"), str(rep), "25"],
                             capture_output=True, text=True).stdout
        lines += ["", "# top SASS lines by warp-stall samples", hot]
        (dst / f"{tag}_ncu_{kern}.txt").write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print("wrote", sorted(p.name for p in dst.iterdir()))


if __name__ == "__main__":
    main()
