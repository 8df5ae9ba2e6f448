"""One batched SPD inverse at the C3 S-inverse shape (for ncu launch lists)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_02090_b200 import _native as nat
lib = nat.load()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
bt, n, b = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (2244, 448, 64)))
X = torch.randn(64, n, n, dtype=torch.float64, device="cuda")
A0 = (X @ X.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device="cuda")).repeat((bt + 63) // 64, 1, 1)[:bt].contiguous()
ws = torch.empty(lib.bddc_spd_inverse_workspace(n, bt, b) // 8 + 2, dtype=torch.float64, device="cuda")
info = torch.zeros(1, dtype=torch.int32, device="cuda")
nat.call("bddc_spd_inverse_batched", nat.ptr(A0), n, n, n * n, bt, b, nat.ptr(ws), nat.ptr(info), st)
torch.cuda.synchronize()
print("ok", int(info.item()))
