"""World-size-2 gloo tests (CPU) of the multi-GPU host plumbing: the
ncclUniqueId bootstrap, the vertex-cyclic ownership, and the max/sum over
ranks used for timing.  The NCCL exchange itself needs GPUs (tests -m gpu run
its single-rank instance)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2003_04920_b200 import dist as pdist
        from paper_2003_04920_b200 import pirrt
        uid = pdist.broadcast_unique_id(pirrt.nccl_unique_id)
        owned = [v for v in range(1001) if pdist.owner(v, world) == rank]
        mx = pdist.max_over_ranks(float(rank + 1))
        sm = pdist.sum_over_ranks(float(len(owned)))
        q.put((rank, uid, owned, mx, sm))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_bootstrap_and_ownership():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    (r0, uid0, own0, mx0, sm0), (r1, uid1, own1, mx1, sm1) = res
    assert len(uid0) == 128 and uid0 == uid1          # every rank got rank 0's id
    assert sorted(own0 + own1) == list(range(1001))    # each vertex owned exactly once
    assert not set(own0) & set(own1)
    assert mx0 == mx1 == 2.0
    assert sm0 == sm1 == 1001.0
