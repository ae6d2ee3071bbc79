"""Matrix-free input: the seeded GENERAL matrix is
decomposed without being stored.  The device computes the same entries as the stored
generator, so the result must be bitwise equal to decomposing the stored matrix; the oracle
(host regeneration of the entries by the independent input module) pins it at sampled
strings where the matrix is too large to store twice."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
from paper_2403_11644_b200 import dist as pdist

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


@pytest.mark.parametrize("n", [1, 4, 7, 9, 11, 13, 15])
def test_generated_bitwise_equals_stored(gpu, n):
    torch = _torch()
    A = ptdr.generate_dense(n, 4, "general")
    ref = ptdr.decompose(A)
    del A
    got = ptdr.decompose_generated(n, 4)
    assert torch.equal(torch.view_as_real(got), torch.view_as_real(ref))
    assert ptdr.last_launch_count() >= 1
    del got, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,world", [(12, 2), (14, 8), (15, 8)])
def test_generated_shards_bitwise(gpu, n, world):
    """Each rank's shard (no communication) == its q-slice of the one-GPU output."""
    torch = _torch()
    ref = ptdr.decompose(ptdr.generate_dense(n, 4, "general"))
    torch.cuda.empty_cache()
    for h in (0, world // 2, world - 1):
        loc = ptdr.decompose_generated(n, 4, h, world)
        idx = torch.from_numpy(pdist.global_q_array(h, n, world)).cuda()
        assert torch.equal(torch.view_as_real(loc), torch.view_as_real(ref[idx])), h
        del loc, idx
    del ref
    torch.cuda.empty_cache()


def test_generated_n16_sampled(gpu):
    """n = 16 without storing the 64 GiB input: sampled coefficients vs the oracle."""
    torch = _torch()
    n = 16
    out = ptdr.decompose_generated(n, 4)
    rng = np.random.default_rng(161)
    qs = np.unique(np.concatenate([rng.integers(0, 4 ** n, 192), [0, 4 ** n - 1]])).astype(np.uint64)
    want = oracle.coeffs_generated(n, 4, 0, qs)
    got = out[torch.from_numpy(qs.astype(np.int64)).cuda()].cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-12 * 6.0
    del out
    torch.cuda.empty_cache()


def test_generated_rejects_small_shards(gpu):
    with pytest.raises(ptdr.PtdrError):
        ptdr.decompose_generated(10, 4, 0, 4)          # n - log2(world) < 11
