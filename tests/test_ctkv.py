"""CTKV format parity with reference-written files (tests/golden/*.ctkv) and the
CTKV -> importance-ordered pool loader (acceptance criterion 11 semantics,
tests/test_acceptance.py:268-295)."""

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2605_24022_b200 import ctkv
from paper_2605_24022_b200.errors import IoError


def test_header_and_round_trip_bytes():
    data = (GOLDEN / "fmt_ranked.ctkv").read_bytes()
    assert data[:4] == b"CTKV"
    assert np.array_equal(np.frombuffer(data[4:32], dtype="<u4"), [1, 4, 32, 2, 8, 0, 1])
    chunk, rk = ctkv.read_ctkv(data, "fmt")
    assert rk is not None and rk.n_layers == 4
    assert ctkv.write_ctkv(chunk, rk) == data          # byte-identical re-serialisation
    bare = (GOLDEN / "fmt_bare.ctkv").read_bytes()
    c2, r2 = ctkv.read_ctkv(bare, "fmt")
    assert r2 is None and ctkv.write_ctkv(c2) == bare
    assert len(data) == ctkv.chunk_file_bytes(4, 32, 2, 8, True)
    assert len(bare) == ctkv.chunk_file_bytes(4, 32, 2, 8, False)


def test_rejects_garbage():
    data = (GOLDEN / "fmt_ranked.ctkv").read_bytes()
    with pytest.raises(IoError):
        ctkv.read_ctkv(b"XXXX" + data[4:])
    with pytest.raises(IoError):
        ctkv.read_ctkv(data[:-3])
    with pytest.raises(IoError):
        ctkv.read_ctkv(data[:10])


@pytest.mark.gpu
def test_pool_from_ctkv_fetch_bit_exact():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    data = (GOLDEN / "fmt_ranked.ctkv").read_bytes()
    chunk, rk = ctkv.read_ctkv(data, "fmt")
    for loc in ("hbm", "pinned"):
        pool = ctkv.pool_from_ctkv([GOLDEN / "fmt_ranked.ctkv"], location=loc,
                                   dtype=torch.float32)
        for r in (0.0, 0.33, 1.0):
            for layer in range(4):
                plan = pool.plan_sparse_fetch("fmt_ranked", layer, r)
                assert plan.expected_bytes == plan.keep_count * 2 * 8 * 4 * 2
                K, V, keep = pool.fetch_sparse(plan)
                if keep.size:
                    assert np.array_equal(K.cpu().numpy(), chunk.keys_raw[layer].data[keep])
                    assert np.array_equal(V.cpu().numpy(), chunk.values[layer].data[keep])
