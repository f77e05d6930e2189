"""World-size-2 gloo tests (CPU) of the multi-GPU host plumbing that
bench.py's sharded leg uses: the ncclUniqueId bootstrap (rank 0's id on
every rank), the rank/world read from the torchrun environment, and the
element-wise max (timing) / sum (relaxation shares) over ranks.  The record
exchange itself runs in libpirrt: on one GPU as in-process rank groups
(tests/test_parity_group_gpu.py), over NCCL with one rank (-m gpu)."""
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
        os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
        env = pdist.env_rank_world()
        uid = pdist.broadcast_unique_id(pirrt.nccl_unique_id)
        mx = pdist.max_over_ranks([float(rank + 1), 10.0 - rank])
        sm = pdist.sum_over_ranks([float(rank + 1), 2.5])
        q.put((rank, uid, env, mx, sm))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_world2_bootstrap_and_reductions():
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
    (r0, uid0, env0, mx0, sm0), (r1, uid1, env1, mx1, sm1) = res
    assert len(uid0) == 128 and uid0 == uid1          # every rank got rank 0's id
    assert env0 == (0, 2, 0) and env1 == (1, 2, 1)
    assert mx0 == mx1 == [2.0, 10.0]                   # element-wise max
    assert sm0 == sm1 == [3.0, 5.0]                    # element-wise sum
