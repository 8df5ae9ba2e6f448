"""Time bddc_gemv on an N x N matrix for each warps-per-row setting."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C, torch
from paper_1901_02090_b200 import _native as nat
lib = nat.load()
for n in [int(v) for v in (sys.argv[1:] or ["2244", "4096", "1000"])]:
    M = torch.randn(n, n, dtype=torch.float64, device="cuda")
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    ref = M @ x
    flush = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for wpr in (1, 2, 4, 8, 0):
        lib.bddc_set_gemv_wpr(wpr)
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        ts = []
        for r in range(30):
            flush.fill_(r)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            lib.bddc_gemv(n, n, n, C.c_void_p(M.data_ptr()), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), st)
            b.record(); b.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
        ts = sorted(ts[5:])
        err = float((y - ref).abs().max() / ref.abs().max())
        print(f"n={n} wpr={wpr} median {ts[len(ts)//2]:.1f} us  min {ts[0]:.1f}  GB/s {8*n*n/ts[len(ts)//2]/1e3:.0f} err {err:.1e}")
    lib.bddc_set_gemv_wpr(0)
