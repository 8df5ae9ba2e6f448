"""Measure the FP64 GEMM ceiling on this B200 (cuBLAS DGEMM via torch) and our DMMA dgemm."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_02090_b200 import _native as nat
nat.load()
out = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a, b, out=c)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 / 1000
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n ** 3 / t / 1e12
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    def ours():
        nat.call("bddc_dgemm_batched", 0, 0, n, n, n, 1.0, nat.ptr(a), n, 0, nat.ptr(b), n, 0, 0.0, nat.ptr(c), n, 0, 1, 0, st)
    for _ in range(3):
        ours()
    e0.record()
    for _ in range(5):
        ours()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 5 / 1000
    out[f"ours_dmma_dgemm_{n}_tflops"] = 2 * n ** 3 / t / 1e12
    ref = a @ b
    out[f"ours_rel_err_{n}"] = float((c - ref).abs().max() / ref.abs().max())
# batched shapes used by the setup: 2244 x (512^3) sweep-like updates
bt, n, k = 2244, 512, 64
A = torch.randn(bt, k, n, dtype=torch.float64, device="cuda")
Bm = torch.randn(bt, k, n, dtype=torch.float64, device="cuda")
Cm = torch.randn(bt, n, n, dtype=torch.float64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
def bat():
    nat.call("bddc_dgemm_batched", 1, 0, n, n, k, -1.0, nat.ptr(A), n, k * n, nat.ptr(Bm), n, k * n, 1.0, nat.ptr(Cm), n, n * n, bt, 0, st)
bat()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); bat(); bat(); bat(); e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 3 / 1000
out["ours_batched_rank64_update_2244x512_tflops"] = 2 * bt * n * n * k / t / 1e12
out["ours_batched_rank64_update_2244x512_GBps"] = bt * (2 * n * n + 2 * k * n) * 8 / t / 1e9
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/fp64_peak.json", "w"), indent=1)
