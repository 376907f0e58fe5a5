"""Request-level data parallelism (BASELINE config 5): replicas only.

Independent RAG requests shard across ranks with NO collective on the hot
path (one process per GPU, torch.distributed over NCCL for plumbing).  After
the timed region one gather collects the per-request results -- first-token
logits, selected index sets, TTFT -- and timings are reduced as the max over
ranks.  The same code runs over gloo on CPU in the tests.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as dist


def world() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_requests(n_requests: int, rank: int, world_size: int) -> list[int]:
    """Request i runs on rank i % world_size (64/G per GPU for config 5)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank/world")
    return list(range(rank, n_requests, world_size))


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over ranks (timing = slowest rank)."""
    rank, ws = world()
    if ws == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


@dataclass
class RequestResult:
    request: int
    ttft_ms: float
    first_token_logits: torch.Tensor   # [vocab] f32
    selected: torch.Tensor             # int32 global recomputed positions


def gather_results(local: list[RequestResult], vocab: int, n_selected: int, device=None):
    """All ranks contribute their request results; rank 0 returns them ordered
    by request id (others return None).  Fixed-size tensors so one all_gather
    per field suffices (NCCL over NVLink on the GPU box, gloo in tests)."""
    rank, ws = world()
    dev = device or (local[0].first_token_logits.device if local else torch.device("cpu"))
    n_local = len(local)
    if ws == 1:
        return sorted(local, key=lambda r: r.request)
    counts = torch.tensor([n_local], dtype=torch.int64, device=dev)
    all_counts = [torch.zeros_like(counts) for _ in range(ws)]
    dist.all_gather(all_counts, counts)
    cap = int(max(c.item() for c in all_counts))
    ids = torch.full((cap,), -1, dtype=torch.int64, device=dev)
    ttft = torch.zeros((cap,), dtype=torch.float64, device=dev)
    logits = torch.zeros((cap, vocab), dtype=torch.float32, device=dev)
    sel = torch.zeros((cap, n_selected), dtype=torch.int32, device=dev)
    for i, r in enumerate(local):
        ids[i] = r.request
        ttft[i] = r.ttft_ms
        logits[i] = r.first_token_logits.to(dev)
        sel[i, : r.selected.numel()] = r.selected.to(dev)
    out = []
    for t in (ids, ttft, logits, sel):
        bufs = [torch.empty_like(t) for _ in range(ws)]
        dist.all_gather(bufs, t)
        out.append(torch.cat(bufs))
    if rank != 0:
        return None
    res = []
    for j in range(out[0].numel()):
        if int(out[0][j]) >= 0:
            res.append(RequestResult(int(out[0][j]), float(out[1][j]), out[2][j], out[3][j]))
    return sorted(res, key=lambda r: r.request)


def gpu_local_cpus(device_index: int) -> list[int] | None:
    """Host CPUs on the NUMA node of CUDA device `device_index` (NVML CPU
    affinity of the device with that PCI bus id), or None when NVML or the
    device is unavailable."""
    try:
        import pynvml
        props = torch.cuda.get_device_properties(device_index)
        bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            n_words = ((os.cpu_count() or 64) + 63) // 64
            mask = pynvml.nvmlDeviceGetCpuAffinity(h, n_words)
        finally:
            pynvml.nvmlShutdown()
    except Exception:  # noqa: BLE001 - advisory only
        return None
    return cpus_from_mask(mask) or None


def cpus_from_mask(mask) -> list[int]:
    """CPU ids set in an NVML affinity mask (64-bit words, CPU 0 = bit 0 of word 0)."""
    return [w * 64 + b for w, word in enumerate(mask) for b in range(64) if (int(word) >> b) & 1]


def bind_to_gpu_numa(device_index: int) -> list[int] | None:
    """Pin this rank's process to the CPUs local to its GPU, so the pinned-host
    chunk pool it allocates next is first-touched on that NUMA node and the
    per-layer sparse H2D copies never cross the inter-socket link (one process
    per GPU; eight pools of 3.65 GB/request each at N = 8).  Returns the CPU
    list, or None (nothing changed) when the affinity cannot be determined."""
    cpus = gpu_local_cpus(device_index)
    if not cpus:
        return None
    try:
        allowed = os.sched_getaffinity(0)
        cpus = [c for c in cpus if c in allowed]
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
    except (AttributeError, OSError):
        return None
    return cpus
