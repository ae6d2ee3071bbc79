"""Batched small matrices (ptdr_decompose_batched_async): every matrix of a batch gives
bitwise the result of decomposing it alone, which the single-matrix tests pin to the
oracle; one matrix per batch is also checked against the oracle directly."""
import numpy as np
import pytest

import oracle
import paper_2403_11644_b200 as ptdr
import ptdr_inputs

pytestmark = pytest.mark.gpu


def _torch():
    import torch

    return torch


@pytest.mark.parametrize("variant", ["general", "hermitian", "real_symmetric"])
@pytest.mark.parametrize("n,batch", [(1, 5), (3, 17), (5, 64), (6, 100), (8, 9), (9, 4), (10, 3)])
def test_batched_equals_single(gpu, n, batch, variant):
    torch = _torch()
    As = np.stack([ptdr_inputs.dense(n, 500 + k, variant) for k in range(batch)])
    A = torch.from_numpy(As).cuda()
    out = ptdr.decompose_batched(A, variant)
    for k in range(batch):
        single = ptdr.decompose(A[k].contiguous(), variant)
        assert torch.equal(torch.view_as_real(out[k]), torch.view_as_real(single)), k
    k = batch // 2
    want = oracle.decompose(As[k])
    assert np.max(np.abs(out[k].cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(As[k]))


def test_batched_rejects_large_n(gpu):
    torch = _torch()
    A = torch.zeros((1, 2048, 2048), dtype=torch.complex128, device="cuda")
    with pytest.raises(ptdr.PtdrError) as e:
        ptdr.decompose_batched(A)
    assert e.value.status == ptdr.PTDR_EINVAL


def test_batched_empty_batch_is_a_noop(gpu):
    torch = _torch()
    A = torch.zeros((0, 64, 64), dtype=torch.complex128, device="cuda")
    out = ptdr.decompose_batched(A)
    assert out.shape == (0, 4 ** 6)
    assert ptdr.last_launch_count() == 0
