import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1812_04315_b200 import _lib, _ops
k = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
P = torch.randn((k, rows), device="cuda")
st = _lib.new_status()
for _ in range(3): _ops.orthonormalize(P, st)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): _ops.orthonormalize(P, st)
b.record(); torch.cuda.synchronize()
print(f"QR k={k} rows={rows}: {a.elapsed_time(b)/20*1e3:.1f} us")
import ctypes, numpy as np
lib = _lib.load_library()
buf = (ctypes.c_ulonglong * 16)()
lib.nenmf_debug_qr_trace.argtypes = [ctypes.c_void_p]
lib.nenmf_debug_qr_trace(ctypes.addressof(buf))
t = np.array(buf[:11], dtype=np.int64)
print("phase us:", np.round(np.diff(t) / 1e3, 2).tolist())
