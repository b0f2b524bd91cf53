"""World-size-2 gloo test of bench.py's multi-process plumbing on CPU (DESIGN.md
sect. 6): rendezvous on 127.0.0.1, barrier, max-over-ranks timing, and the z-slab
split of ONE lattice over the ranks.  No GPU, no CUDA extension."""
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
    from paper_math_0508111_b200 import slab
    cfg = CONFIGS[1]
    assert f"sharded over {ws} ranks" in bench.workload_config(cfg, w)["parallelism"]
    L = 6
    z0, nz = slab.slab_bounds(L, rank, ws)
    eps = an.disorder(L, cfg["W"], cfg["seed"])[z0 * L * L:(z0 + nz) * L * L]   # this rank's slab
    out.put((rank, m, (z0, nz), float(eps.sum())))
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
    assert s0 == (0, 3) and s1 == (3, 3)   # the two slabs tile the lattice
    from inputs import CONFIGS
    from oracle import anderson as an
    cfg = CONFIGS[1]
    assert np.isclose(e0 + e1, an.disorder(6, cfg["W"], cfg["seed"]).sum(), rtol=0, atol=1e-12)


def _halo_worker(rank, ws, port, L, out):
    os.environ.update(WORLD_SIZE=str(ws), RANK=str(rank), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_math_0508111_b200 import slab
    dist.init_process_group("gloo")
    z0, nz = slab.slab_bounds(L, rank, ws)
    P = L * L
    full = torch.arange(L * P, dtype=torch.float64)        # x_s = s: every plane is identifiable
    x_ext = torch.full(((nz + 2) * P,), -1.0, dtype=torch.float64)
    x_ext[P:(nz + 1) * P] = full[z0 * P:(z0 + nz) * P]
    slab.halo_exchange(x_ext, L, nz)
    lo_ok = torch.equal(x_ext[:P], full[((z0 - 1) % L) * P:((z0 - 1) % L + 1) * P])
    hi_ok = torch.equal(x_ext[(nz + 1) * P:], full[((z0 + nz) % L) * P:((z0 + nz) % L + 1) * P])
    out.put((rank, z0, nz, bool(lo_ok), bool(hi_ok)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("ws,L", [(2, 5), (3, 7)])
def test_slab_halo_exchange(ws, L):
    # z-slab sharding (row (e)): uneven slab bounds cover the lattice; every rank's halo
    # planes are its periodic neighbours' boundary planes after one exchange
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, ws, port, L, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(nz for _, _, nz, _, _ in res) == L
    assert [z0 for _, z0, _, _, _ in res] == sorted(z0 for _, z0, _, _, _ in res)
    assert all(lo and hi for _, _, _, lo, hi in res)


def test_slab_bounds_and_single_rank_halo():
    import torch
    sys.path.insert(0, ROOT)
    from paper_math_0508111_b200 import slab
    assert [slab.slab_bounds(10, r, 3) for r in range(3)] == [(0, 4), (4, 3), (7, 3)]
    L, P = 4, 16
    x = torch.arange(L * P, dtype=torch.float64)
    xe = torch.cat([torch.zeros(P, dtype=torch.float64), x, torch.zeros(P, dtype=torch.float64)])
    slab.halo_exchange(xe, L, L)                     # one rank: periodic wrap
    assert torch.equal(xe[:P], x[(L - 1) * P:]) and torch.equal(xe[(L + 1) * P:], x[:P])


def _comm_worker(rank, ws, port, L, out):
    # the tensor-level core of slab.TorchComm (the aj_comm the sharded solve calls):
    # sum / max all-reduce and the periodic plane exchange, on the default group and on a
    # subgroup (P2P peers are global ranks)
    os.environ.update(WORLD_SIZE=str(ws), RANK=str(rank), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_math_0508111_b200 import slab
    dist.init_process_group("gloo")
    res = {}
    c = slab.TorchComm()
    t = torch.tensor([1.0 + rank, -2.0 * rank, 0.5], dtype=torch.float64)
    c.allreduce_(t, 0)
    res["sum"] = t.tolist()
    t = torch.tensor([float(rank), -float(rank)], dtype=torch.float64)
    c.allreduce_(t, 1)
    res["max"] = t.tolist()
    z0, nz = slab.slab_bounds(L, rank, ws)
    P = L * L
    full = torch.arange(L * P, dtype=torch.float64)
    mine = full[z0 * P:(z0 + nz) * P]
    lo, hi = torch.empty(P, dtype=torch.float64), torch.empty(P, dtype=torch.float64)
    c.exchange_(mine[:P], mine[(nz - 1) * P:], lo, hi)
    res["halo"] = (bool(torch.equal(lo, full[((z0 - 1) % L) * P:((z0 - 1) % L + 1) * P])),
                   bool(torch.equal(hi, full[((z0 + nz) % L) * P:((z0 + nz) % L + 1) * P])))
    # subgroup of the odd-or-even ranks: its own slabs, halos among its members only
    members = [r for r in range(ws) if r % 2 == 0]
    grp = dist.new_group(members)
    if rank in members:
        gc = slab.TorchComm(grp)
        gw, gr = len(members), members.index(rank)
        z0, nz = slab.slab_bounds(L, gr, gw)
        mine = full[z0 * P:(z0 + nz) * P]
        c.__class__.exchange_(gc, mine[:P], mine[(nz - 1) * P:], lo, hi)
        res["sub"] = (bool(torch.equal(lo, full[((z0 - 1) % L) * P:((z0 - 1) % L + 1) * P])),
                      bool(torch.equal(hi, full[((z0 + nz) % L) * P:((z0 + nz) % L + 1) * P])))
        s = torch.tensor([1.0], dtype=torch.float64)
        gc.allreduce_(s)
        res["subsum"] = float(s.item())
    out.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("ws,L", [(2, 6), (3, 7), (4, 9)])
def test_torch_comm_core(ws, L):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, ws, port, L, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(ws):
        assert res[r]["sum"] == [sum(1.0 + k for k in range(ws)), sum(-2.0 * k for k in range(ws)), 0.5 * ws]
        assert res[r]["max"] == [ws - 1.0, 0.0]
        assert res[r]["halo"] == (True, True)
    members = [r for r in range(ws) if r % 2 == 0]
    for r in members:
        assert res[r]["sub"] == (True, True)
        assert res[r]["subsum"] == float(len(members))
