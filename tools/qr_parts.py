"""Time the CholeskyQR2 stages separately (nenmf_panel_* entry points)."""
import sys, ctypes
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib
lib = _lib.load_library()
k = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
P = torch.randn((k, rows), device="cuda")
Q = torch.empty_like(P)
G = torch.empty((k, k), dtype=torch.float64, device="cuda")
R = torch.empty((k, k), dtype=torch.float64, device="cuda")
meta = torch.empty(k + 4, dtype=torch.int32, device="cuda")
st = _lib.new_status()
ws = _lib.workspace(lib.nenmf_panel_gram_workspace_bytes(1, rows, k))
s = _lib.stream_handle()
def gram(): lib.nenmf_panel_gram(1, P.data_ptr(), rows, k, G.data_ptr(), ws.data_ptr(), ws.numel(), s)
def fac(): lib.nenmf_panel_factor(G.data_ptr(), k, 1, R.data_ptr(), meta.data_ptr(), _lib.status_ptr(st), s)
def fac0(): lib.nenmf_panel_factor(G.data_ptr(), k, 0, R.data_ptr(), meta.data_ptr(), _lib.status_ptr(st), s)
def trsm(): lib.nenmf_panel_trsm(1, P.data_ptr(), rows, k, R.data_ptr(), meta.data_ptr(), Q.data_ptr(), 0, 0, s)
for name, fn in [("gram+reduce", gram), ("factor pivoted", fac), ("factor plain", fac0), ("trsm", trsm)]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): fn()
    b.record(); torch.cuda.synchronize()
    print(f"{name:16s} {a.elapsed_time(b)/50*1e3:7.1f} us", flush=True)
print("rank", int(meta[0]))
