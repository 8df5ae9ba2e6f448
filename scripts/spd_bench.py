"""Batched SPD inverse throughput (flops = n^3 per matrix) for the setup shapes.
regs: 3 = register leaves + split 64-leaf, 1 = register leaves, 0 = shared-memory leaves."""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_02090_b200 import _native as nat
lib = nat.load()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
res = {}
import itertools
shapes = [(2244, 512), (2244, 448), (2244, 160), (2244, 32), (1, 2304)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1].split(",")]
leaves = (32, 64) if len(sys.argv) > 1 else (64,)
for (bt, n), regs in itertools.product(shapes, (3, 1, 0) if len(sys.argv) <= 1 else (3, 1)):
    lib.bddc_set_leaf_regs(regs)
    for b in leaves:
        if n % b:
            continue
        X = torch.randn(min(bt, 64), n, n, dtype=torch.float64, device="cuda")
        A0 = X @ X.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device="cuda")
        A0 = A0.repeat((bt + 63) // 64, 1, 1)[:bt].contiguous()
        M = A0.clone()
        ws = torch.empty(lib.bddc_spd_inverse_workspace(n, bt, b) // 8 + 2, dtype=torch.float64, device="cuda")
        info = torch.zeros(1, dtype=torch.int32, device="cuda")
        def run():
            M.copy_(A0)
            nat.call("bddc_spd_inverse_batched", nat.ptr(M), n, n, n * n, bt, b, nat.ptr(ws), nat.ptr(info), st)
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(); M.copy_(A0); e3.record()
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        t = (e0.elapsed_time(e1) - e2.elapsed_time(e3)) / 1000
        err = float((M[0] @ A0[0] - torch.eye(n, dtype=torch.float64, device="cuda")).abs().max())
        res[f"{bt}x{n} b={b} regs={regs}"] = dict(ms=round(t * 1000, 3), tflops=round(bt * n ** 3 / t / 1e12, 2), err=err)
        print(f"{bt}x{n} b={b} regs={regs}: {t*1000:.2f} ms  {bt*n**3/t/1e12:.2f} TF/s  |MA-I|={err:.1e}", flush=True)
if len(sys.argv) <= 1:
    json.dump(res, open("gpurun_out/spd_bench.json", "w"), indent=1)
