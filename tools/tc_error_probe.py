"""Locate the error structure of the tcgen05 attention vs an fp32 reference."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2605_24022_b200 import _dev, _lib
torch.manual_seed(0)
A, HQ, HKV, D, N = 512, 32, 8, 128, 4096
gen = torch.Generator(device="cuda").manual_seed(1)
scale_q = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
q = (scale_q * torch.randn((A, HQ, D), device="cuda", generator=gen)).to(torch.bfloat16)
k = torch.randn((N, HKV, D), device="cuda", generator=gen).to(torch.bfloat16)
v = torch.randn((N, HKV, D), device="cuda", generator=gen).to(torch.bfloat16)
pos = torch.sort(torch.randperm(N, device="cuda", generator=gen)[:A])[0].to(torch.int32)
out = torch.empty_like(q)
_lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(pos), A, HQ, _dev.ptr(k), _dev.ptr(v), N, HKV, D, HKV*D, 1/D**0.5, 1, _dev.ptr(out), 1, None, None, 0, _dev.stream_handle())
kk = k.float().repeat_interleave(4, 1).permute(1, 2, 0); vv = v.float().repeat_interleave(4, 1).permute(1, 0, 2)
s = torch.bmm(q.float().permute(1, 0, 2), kk) / D**0.5
mask = torch.arange(N, device="cuda")[None, :] <= pos[:, None].long()
s = s.masked_fill(~mask[None], float("-inf"))
m = s.amax(-1, keepdim=True); p = torch.exp(s - m); l = p.sum(-1, keepdim=True)
ref = (torch.bmm(p, vv) / l).permute(1, 0, 2)
emu = (torch.bmm(p.to(torch.bfloat16).float(), vv) / l).permute(1, 0, 2)
err = (out.float() - ref).abs().amax(-1)  # [A, HQ]
erre = (emu - ref).abs().amax(-1)
print("scale_q", scale_q, "max|ref|", ref.abs().max().item(), "kernel max err", err.max().item(), "emu max err", erre.max().item())
idx = torch.topk(err.flatten(), 10).indices
for i in idx.tolist():
    a, h = divmod(i, HQ)
    print(f"a={a} (a%32={a%32}) h={h} pos={pos[a].item()} err={err[a,h].item():.4f} emu={erre[a,h].item():.4f} nb={pos[a].item()//128+1} rowmax_p_frac={(p[h,a].max()/l[h,a,0]).item():.3f}")
# repeatability
out2 = torch.empty_like(q)
_lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(pos), A, HQ, _dev.ptr(k), _dev.ptr(v), N, HKV, D, HKV*D, 1/D**0.5, 1, _dev.ptr(out2), 1, None, None, 0, _dev.stream_handle())
print("run-to-run max diff", (out2.float()-out.float()).abs().max().item())
