"""world_size-2 gloo test of the replica harness bench.py uses for N > 1."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    from paper_1801_08464_b200.replicas import Replicas
    from paper_1801_08464_b200 import synth
    r = Replicas("gloo")
    s = synth.make_config(2, 6, seed=r.seed())
    r.barrier()
    t = r.max(10.0 + rank)
    tot = r.sum(s.n)
    q.put((rank, t, tot, float(s.rhs[0])))
    r.close()


def test_two_rank_replicas():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(t == 11.0 for _, t, _, _ in res)          # max over ranks
    assert all(tot == 2 * 432 for _, _, tot, _ in res)   # whole-job DOFs
    assert res[0][3] != res[1][3]                         # independent systems per replica
    assert np.isfinite([x[3] for x in res]).all()
