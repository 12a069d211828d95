"""The device input generator (coot_fill) reproduces the oracle's generator
bit for bit (both implement the recipe independently)."""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, requires_gpu, to_host
from progs import ALL

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.fixture(scope="module")
def ctx():
    import paper_2508_11385_b200 as coot
    return coot.Context(0)


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("kind", ["randu", "ones", "iota", "modk", "colidx", "rowidx", "zeros"])
def test_fill_matches_oracle(ctx, etype, kind):
    n, start, m = 300_007, 12345, 977
    t = torch.empty(n, dtype=TORCH[etype], device="cuda")
    ctx.fill(t, kind, seed=42, stream=3, start=start, n_rows=m, k=13)
    torch.cuda.synchronize()
    want = oracle.fill(etype, kind, n, seed=42, stream=3, start=start, n_rows=m, k=13)
    got = to_host(t, etype)
    assert np.array_equal(got.view(np.uint8), want.view(np.uint8))


def test_fill_vigna_first_outputs(ctx):
    t = torch.empty(3, dtype=torch.int64, device="cuda")
    ctx.fill(t, "randu", seed=0, stream=0)
    torch.cuda.synchronize()
    got = [int(x) & (2**64 - 1) for x in t.cpu().tolist()]
    assert got == [0xe220a8397b1dcdaf, 0x6e789e6aa1b965f4, 0x06c45d188009454f]
