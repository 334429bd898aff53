"""N>1 path on CPU: world_size-2 gloo processes each take their contiguous
shard (vd_shard_range) of the same seeded batch, evaluate it (the CPU oracle
stands in for the kernels here, there is no GPU), and the rank-ordered gather
is bit-identical to the single-process evaluation — the sharding contract of
DESIGN.md §Multi-GPU (no data-path collective)."""
import os
import socket
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, N, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_ffi
    from paper_2604_04310_b200 import dist as vdist

    om = oracle_ffi.Model.builtin("chain7")
    b, e = vdist.local_shard(N)
    qq, qd, qdd, _ = om.random_states(N, 2604, True, False)
    local = torch.as_tensor(om.rnea(qq[b:e], qd[b:e], qdd[b:e], threads=1))
    t = vdist.max_over_ranks(float(rank + 1))
    full = vdist.gather_rows(local, N)
    if rank == 0:
        q.put((full.numpy(), t, (b, e)))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_concatenate_bit_identically(oracle):
    N = 1001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax, span0 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    om = oracle.Model.builtin("chain7")
    qq, qd, qdd, _ = om.random_states(N, 2604, True, False)
    ref = om.rnea(qq, qd, qdd, threads=1)
    assert np.array_equal(full, ref)
    assert tmax == 2.0
    assert span0 == (0, 501)
