import sys, time, subprocess
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2605_24022_b200 as ct
from paper_2605_24022_b200.spectral import score_device, score_select_fast
cfg = ct.ModelConfig.llama3_8b(n_layers=32, seed=1234)
model = ct.GpuModel.random(cfg, dtype=torch.bfloat16)
rng = np.random.default_rng([0, 7])
chunks = [ct.encode_chunk_isolated(model, rng.integers(0, cfg.vocab_size, size=2048), chunk_id=f"c{j}") for j in range(16)]
keys = torch.stack([c.keys for c in chunks]); vals = torch.stack([c.values for c in chunks])
def clk():
    return subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active","--format=csv,noheader"],capture_output=True,text=True).stdout.strip()
for name, fn in (("f64", lambda: score_device(keys, vals, 0.5, "f64", want_layer_order=False)), ("fast", lambda: score_select_fast(keys, vals, 308)), ("fast", lambda: score_select_fast(keys, vals, 308))):
    for i in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); t0=time.perf_counter()
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        print(name, i, f"{s.elapsed_time(e):.2f} ms (wall {1e3*(time.perf_counter()-t0):.2f})", clk(), flush=True)
