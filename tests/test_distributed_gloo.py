"""Config-5 sharding on CPU: world_size 2 over gloo (127.0.0.1).  Requests are
sharded with no hot-path collective; results and max-over-ranks timings are
gathered afterwards exactly as bench.py does over NCCL."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_24022_b200.distributed import (RequestResult, gather_results, max_over_ranks,
                                               shard_requests)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world_size, port, n_req, vocab, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world_size)
    try:
        mine = shard_requests(n_req, rank, world_size)
        local = []
        for i in mine:
            g = torch.Generator().manual_seed(i)
            local.append(RequestResult(i, 10.0 + i, torch.randn(vocab, generator=g),
                                       torch.arange(i, i + 5, dtype=torch.int32)))
        t = max_over_ranks(1.0 + rank)
        res = gather_results(local, vocab, 5)
        if rank == 0:
            q.put((t, [(r.request, r.ttft_ms, float(r.first_token_logits.sum()),
                        r.selected.tolist()) for r in res]))
    finally:
        dist.destroy_process_group()


def test_shard_requests_partition():
    for ws in (1, 2, 4, 8):
        seen = sorted(i for r in range(ws) for i in shard_requests(64, r, ws))
        assert seen == list(range(64))
        assert all(len(shard_requests(64, r, ws)) == 64 // ws for r in range(ws))


@pytest.mark.timeout(120)
def test_gather_and_max_over_two_gloo_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_req, vocab = 7, 33
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_req, vocab, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, res = q.get(timeout=100)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    assert t == 2.0  # max over ranks
    assert [r[0] for r in res] == list(range(n_req))
    for i, ttft, lsum, sel in res:
        g = torch.Generator().manual_seed(i)
        assert ttft == 10.0 + i
        assert abs(lsum - float(torch.randn(vocab, generator=g).sum())) < 1e-5
        assert sel == list(range(i, i + 5))


def test_numa_mask_decode_and_safe_bind():
    from paper_2605_24022_b200.distributed import bind_to_gpu_numa, cpus_from_mask
    assert cpus_from_mask([0b1011, 0]) == [0, 1, 3]
    assert cpus_from_mask([0, 1 << 63, 1]) == [127, 128]
    assert cpus_from_mask([]) == []
    if not torch.cuda.is_available():  # no device: nothing is changed
        before = os.sched_getaffinity(0)
        assert bind_to_gpu_numa(0) is None
        assert os.sched_getaffinity(0) == before
