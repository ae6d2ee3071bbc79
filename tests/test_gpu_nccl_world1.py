"""The multi-GPU dense path through a real NCCL process group on the one GPU a test box has
(world_size 1): generate_sendblocks with K sub-ranges -> dist.decompose_sharded (the K
asynchronous all_to_all_singles on NCCL's stream, each sub-range decomposed as soon as its
exchange has landed) -> bitwise the one-GPU decomposition at the positions global_q_sub
names.  With one rank the all-to-all is a local copy, but every call of the N > 1 bench
path runs: process group, NCCL collectives, stream ordering, virtual-rank kernels."""
import socket

import numpy as np
import pytest

import paper_2403_11644_b200 as ptdr
from paper_2403_11644_b200 import dist as pdist

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,K", [(13, 4), (12, 2), (15, 4)])
def test_decompose_sharded_over_nccl_world1(gpu, n, K):
    import torch
    import torch.distributed as dist

    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        ref = ptdr.decompose(ptdr.generate_dense(n, 4, "general"))
        send = ptdr.generate_sendblocks(n, 4, 0, 1, subranges=K)
        side = torch.cuda.Stream()
        out = pdist.decompose_sharded(send, n, stream=side)   # kernels on a non-current stream
        torch.cuda.synchronize()
        assert out.shape == (K, 4 ** n // K)
        w = 2 * (n - (K.bit_length() - 1))
        g = K.bit_length() - 1
        for s in range(K):
            # sub-output s = virtual rank s of world K: block zt holds q_of(s, zt, g) << w ...
            for zt in range(K):
                q0 = ptdr.q_of(s, zt, g) << w
                assert torch.equal(torch.view_as_real(out[s, zt << w:(zt + 1) << w]),
                                   torch.view_as_real(ref[q0:q0 + (1 << w)])), (s, zt)
        # ... and global_q_sub agrees with that block structure
        rng = np.random.default_rng(n)
        for s in range(K):
            for li in rng.integers(0, 4 ** n // K, 8):
                q = pdist.global_q_sub(0, s, int(li), n, 1, K)
                assert torch.equal(torch.view_as_real(out[s, int(li)]), torch.view_as_real(ref[q]))
    finally:
        dist.destroy_process_group()
