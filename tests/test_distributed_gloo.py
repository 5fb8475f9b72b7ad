"""N>1 path on CPU: two processes, gloo backend, 127.0.0.1 rendezvous.  Each rank computes its contiguous
block (CPU oracle through the compute hook) and the heights are gathered with all_gather -- the same
code path bench.py / heights_sharded take under NCCL on GPUs."""
import os
import socket

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, count, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    import oracle
    from paper_2502_12428_b200.distributed import heights_sharded, rank_block
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    z = np.load(os.path.join(GOLDEN, "heights_p3_seed0_w0_3000.npz"))
    coeffs = z["coeffs"][:count]
    seen = []

    def compute(p, c, bound, device):
        seen.append(len(c))
        return oracle.heights_batch(c, p, bound)

    hs, its = heights_sharded(3, coeffs, 10, compute=compute)
    n_mine = rank_block(count, rank, world)[1]
    assert seen == ([n_mine] if n_mine else [])  # an empty block never reaches the engine
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), hs=hs, its=its)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("count", [101, 1])
def test_two_rank_sharding_gloo(tmp_path, count):
    import torch.multiprocessing as mp
    world, port = 2, _free_port()
    mp.spawn(_worker, args=(world, port, count, str(tmp_path)), nprocs=world, join=True)
    z = np.load(os.path.join(GOLDEN, "heights_p3_seed0_w0_3000.npz"))
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(got["hs"], z["heights"][:count]) and np.array_equal(got["its"], z["iters"][:count])
