import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2605_24022_b200 as ct
from oracle import cachetune_oracle as O
cfg = ct.ModelConfig.llama3_8b(n_layers=2, vocab_size=2048, seed=1)
gm = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
rng = np.random.default_rng(2)
toks = [rng.integers(0, 2048, size=2048) for _ in range(2)]
suffix = rng.integers(0, 2048, size=64)
chunks = [ct.encode_chunk_isolated(gm, t, chunk_id=f"c{j}") for j, t in enumerate(toks)]
ranks = [ct.rank_chunk(c) for c in chunks]
res = ct.selective_prefill(gm, chunks, ranks, suffix, 0.15, logits_rows="last")
w = gm.to_numpy_weights()
ocfg = O.ModelConfig(seed=1, n_layers=2, n_heads=32, head_dim=128, vocab_size=2048, mlp="swiglu", n_kv_heads=8, intermediate=14336)
om = O.Model(ocfg, weights=w)
och = [([c.keys[l].float().cpu().numpy() for l in range(2)], [c.values[l].float().cpu().numpy() for l in range(2)], t) for c, t in zip(chunks, toks)]
aggs = [O.rank_chunk(kr, vs)[2] for kr, vs, _ in och]
want = O.selective_prefill(om, och, aggs, suffix, 0.15, want_probs=False, logits_rows="last")
print("logits", O.normwise_rel(res.logits.double().cpu().numpy(), want["logits"]))
rec = want["query_positions"]
for l in range(2):
    K, V = res.kv[l]
    K = K.float().cpu().numpy(); V = V.float().cpu().numpy()
    print(l, "K", O.normwise_rel(K, want["kv"][l][0]), "V", O.normwise_rel(V, want["kv"][l][1]),
          "Krec", O.normwise_rel(K[rec], want["kv"][l][0][rec]), "max|K|", np.abs(want["kv"][l][0]).max(),
          "mean rel err rec", np.mean(np.abs(K[rec]-want["kv"][l][0][rec]))/np.mean(np.abs(want["kv"][l][0][rec])))
# same request with the SIMT fp32-P attention path (probs requested forces it)
res2 = ct.selective_prefill(gm, chunks, ranks, suffix, 0.15, logits_rows="last", record_attention=True)
print("SIMT-attention logits", O.normwise_rel(res2.logits.double().cpu().numpy(), want["logits"]))
for l in range(2):
    K, V = res2.kv[l]
    print(l, "SIMT K", O.normwise_rel(K.float().cpu().numpy(), want["kv"][l][0]), "V", O.normwise_rel(V.float().cpu().numpy(), want["kv"][l][1]))
# attention kernel alone on layer-1 inputs: TC vs fp32 torch
from paper_2605_24022_b200 import _dev, _lib
K1, V1 = res.kv[1]
gen = torch.Generator(device="cuda").manual_seed(0)
A = len(rec); q = torch.randn((A, 32, 128), device="cuda", generator=gen).to(torch.bfloat16)
pos = torch.as_tensor(rec.astype(np.int32), device="cuda")
out = torch.empty_like(q)
_lib.call("ct_selective_attention", _dev.ptr(q), _dev.ptr(pos), A, 32, _dev.ptr(K1), _dev.ptr(V1), K1.shape[0], 8, 128, 8*128, 1/128**0.5, 1, _dev.ptr(out), 1, None, None, 0, _dev.stream_handle())
kk = K1.float().repeat_interleave(4, 1).permute(1, 2, 0); vv = V1.float().repeat_interleave(4, 1).permute(1, 0, 2)
s = torch.bmm(q.float().permute(1, 0, 2), kk) / 128**0.5
mask = torch.arange(K1.shape[0], device="cuda")[None, :] <= pos[:, None].long()
s = s.masked_fill(~mask[None], float("-inf"))
ref = torch.bmm(torch.softmax(s, -1), vv).permute(1, 0, 2)
print("TC attention vs fp32 torch: normwise", ((out.float()-ref).abs().max()/ref.abs().max()).item(), "mean rel", ((out.float()-ref).abs().mean()/ref.abs().mean()).item())
# emulate bf16-rounded P (fp32 exp, fp32 row sum) in torch: does the kernel match it?
m = s.amax(-1, keepdim=True)
p = torch.exp(s - m)
l = p.sum(-1, keepdim=True)
emu = (torch.bmm(p.to(torch.bfloat16).float(), vv) / l).permute(1, 0, 2)
print("bf16-P emulation vs fp32:", ((emu-ref).abs().max()/ref.abs().max()).item(),
      " TC vs emulation:", ((out.float()-emu).abs().max()/ref.abs().max()).item())
emu16 = (torch.bmm(p.half().float(), vv) / l).permute(1, 0, 2)
print("fp16-P emulation vs fp32:", ((emu16-ref).abs().max()/ref.abs().max()).item())
