"""World-size-2 gloo test of bench.py's multi-process plumbing on CPU (DESIGN.md
sect. 6): rendezvous on 127.0.0.1, barrier, max-over-ranks timing, and one
independent disorder realisation per rank.  No GPU, no CUDA extension."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(WORLD_SIZE=str(ws), RANK=str(rank), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist
    from inputs import CONFIGS
    from oracle import anderson as an
    w, r, _ = bench.dist_setup(None)
    assert (w, r) == (ws, rank) and dist.get_backend() == "gloo"
    bench.barrier(w)
    m = bench.allreduce_max(w, 10.0 * (rank + 1))
    seed = bench.replica_seed(CONFIGS[1], rank)
    eps = an.disorder(6, 16.5, seed)
    out.put((rank, m, seed, float(eps.sum())))
    bench.barrier(w)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_bench_plumbing_world_size_2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, m0, s0, e0), (r1, m1, s1, e1) = res
    assert m0 == m1 == 20.0           # max over ranks reaches every rank
    assert s1 == s0 + 1               # distinct realisations per rank
    assert not np.isclose(e0, e1)
