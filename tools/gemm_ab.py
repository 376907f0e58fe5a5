"""cuBLAS vs cuBLASLt (torch preferred_blas_library) on the config-2 step GEMM
shapes; measured mixed (QKV/O faster with Lt, gate-up/down slower), so the
step keeps the default library."""
import torch, time
torch.manual_seed(0)
shapes = {"qkv": (4992, 4096, 6144), "o": (4992, 4096, 4096), "gateup": (4992, 4096, 28672), "down": (4992, 14336, 4096)}
def bench(lib):
    torch.backends.cuda.preferred_blas_library(lib)
    out = {}
    for name, (m, k, n) in shapes.items():
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
        for _ in range(5): torch.mm(a, b)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50): torch.mm(a, b)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 50
        out[name] = (ms, 2 * m * k * n / ms / 1e9)
    return out
for rep in range(2):
    for lib in ("cublas", "cublaslt"):
        r = bench(lib)
        print(lib, {k: f"{v[0]*1e3:.0f}us {v[1]:.0f}TF" for k, v in r.items()})
