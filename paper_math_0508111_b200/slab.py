"""z-slab sharding of the lattice over torch.distributed ranks (row (e); north star:
"the lattice shards naturally into z-slabs across 1/2/4/8 GPUs ... with one-plane
halo exchange and dot-product allreduce via NCCL"; DESIGN.md sect. 6).

Argument marshalling and communication plumbing only: every step of the sharded
solve runs in the CUDA library (jd_solve_sharded / spmv_sharded /
precond_setup_slab), which calls an `aj_comm` (include/anderson_jd.h) for its
cross-rank steps.  Two implementations:

* `nccl_comm()` -- the production one: the library's own NCCL communicator
  (aj_comm_nccl_create; ncclAllReduce on the solve's stream, the halo planes as
  one ncclSend/ncclRecv group on a side stream overlapped with the interior
  planes).  The 128-byte ncclUniqueId travels over torch.distributed.
* `TorchComm` -- the same callbacks over torch.distributed with host staging
  (gloo): used by the tests, where several ranks share one GPU or none.

Layout of a rank's data: planes z0 <= k < z0 + nz of the L^3 lattice, site order of
the full lattice (x fastest), offset z0 L^2.
"""
import ctypes


def slab_bounds(L, rank, world):
    """(z0, nz) of `rank`: contiguous planes, the first L % world ranks one plane more."""
    if not (1 <= world <= L and 0 <= rank < world):
        raise ValueError("need 1 <= world <= L and 0 <= rank < world")
    base, extra = divmod(L, world)
    nz = base + (1 if rank < extra else 0)
    z0 = rank * base + min(rank, extra)
    return z0, nz


def _peers(group):
    """(rank, world, global rank below, global rank above) of this process in `group`
    (P2P peers are global ranks; `down`/`up` are the periodic z neighbours)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    down, up = (rank - 1) % world, (rank + 1) % world
    if group is not None:
        down, up = dist.get_global_rank(group, down), dist.get_global_rank(group, up)
    return rank, world, down, up


def exchange_planes(send_lo, send_hi, recv_lo, recv_hi, group=None):
    """Periodic one-plane halo exchange between z-neighbours: this slab's first plane
    (send_lo) goes to the rank below, its last plane (send_hi) to the rank above;
    recv_lo <- the lower neighbour's last plane, recv_hi <- the upper neighbour's first.
    Tensors on the process group's device (CPU for gloo)."""
    import torch.distributed as dist
    if not dist.is_initialized():  # one process: the periodic wrap
        recv_lo.copy_(send_hi)
        recv_hi.copy_(send_lo)
        return
    rank, world, down, up = _peers(group)
    if world == 1:
        recv_lo.copy_(send_hi)
        recv_hi.copy_(send_lo)
        return
    # posting order matters when down == up (two ranks): messages between a pair are
    # matched in order, so every rank sends (last -> up) before (first -> down) and
    # receives (lower halo <- down) before (upper halo <- up)
    ops = [dist.P2POp(dist.isend, send_hi.contiguous(), up, group),
           dist.P2POp(dist.isend, send_lo.contiguous(), down, group),
           dist.P2POp(dist.irecv, recv_lo, down, group), dist.P2POp(dist.irecv, recv_hi, up, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def halo_exchange(x_ext, L, nz, group=None):
    """Fill the two halo planes of x_ext = [halo below | nz planes | halo above]."""
    P = L * L
    exchange_planes(x_ext[P:2 * P], x_ext[nz * P:(nz + 1) * P], x_ext[:P], x_ext[(nz + 1) * P:(nz + 2) * P], group)
    return x_ext


def spmv_sharded_ext(y, x_ext, eps, L, nz, hop, sigma=0.0, group=None):
    """y = (A - sigma I) x on this rank's slab from an extended vector: halo exchange, then
    the slab stencil kernel (spmv_slab)."""
    from . import binding
    halo_exchange(x_ext, L, nz, group)
    return binding.spmv_slab(y, x_ext, eps, L, nz, hop, sigma)


# --------------------------------------------------------------------------- aj_comm
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_void_p)
HALO_START_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p)
HALO_WAIT_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)


class AjComm(ctypes.Structure):
    """struct aj_comm of include/anderson_jd.h."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("ctx", ctypes.c_void_p),
                ("allreduce", ALLREDUCE_FN), ("halo_start", HALO_START_FN), ("halo_wait", HALO_WAIT_FN)]


class _DevArray:
    """Zero-copy torch view of library-owned device memory (__cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _dev(ptr, n):
    import torch
    return torch.as_tensor(_DevArray(ptr, n), device="cuda")


class TorchComm:
    """aj_comm over torch.distributed with host staging: the stream is synchronised,
    values go through CPU tensors and the process group (gloo), the results are copied
    back.  Plumbing for tests (several ranks on one GPU); the product path is nccl_comm().
    The tensor-level methods `allreduce_` / `exchange_` are the testable core."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._cb = (ALLREDUCE_FN(self._c_allreduce), HALO_START_FN(self._c_halo_start), HALO_WAIT_FN(self._c_wait))
        self.c = AjComm(self.world, self.rank, None, *self._cb)
        self.errors = []

    # ---- core (device-agnostic tensors)
    def allreduce_(self, t, op=0):
        import torch.distributed as dist
        h = t.detach().to("cpu", copy=True)
        dist.all_reduce(h, op=dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM, group=self.group)
        t.copy_(h)
        return t

    def exchange_(self, send_lo, send_hi, recv_lo, recv_hi):
        import torch
        cpu = [t.detach().to("cpu", copy=True) for t in (send_lo, send_hi)]
        rl, rh = torch.empty_like(cpu[0]), torch.empty_like(cpu[1])
        exchange_planes(cpu[0], cpu[1], rl, rh, self.group)
        recv_lo.copy_(rl)
        recv_hi.copy_(rh)

    # ---- C callbacks
    def _sync(self, stream):
        import torch
        torch.cuda.ExternalStream(stream).synchronize() if stream else torch.cuda.synchronize()

    def _c_allreduce(self, ctx, buf, count, op, stream):
        try:
            self._sync(stream)
            self.allreduce_(_dev(buf, count), op)
            return 0
        except Exception as e:  # reported to the caller as a failed callback
            self.errors.append(repr(e))
            return 2

    def _c_halo_start(self, ctx, slo, shi, rlo, rhi, count, stream):
        try:
            self._sync(stream)
            self.exchange_(_dev(slo, count), _dev(shi, count), _dev(rlo, count), _dev(rhi, count))
            return 0
        except Exception as e:
            self.errors.append(repr(e))
            return 2

    def _c_wait(self, ctx, stream):
        return 0

    def ptr(self):
        return ctypes.pointer(self.c)


class NcclComm:
    """The library's NCCL communicator over the ranks of `group` (collective)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        from . import binding
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        path = nccl_library_path()
        uid = torch.zeros(128, dtype=torch.uint8)
        if self.rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            binding._check(binding.lib().aj_nccl_unique_id(path, buf))
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        uid = uid.to(dev)
        dist.broadcast(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        raw = (ctypes.c_uint8 * 128)(*uid.cpu().tolist())
        self.h = ctypes.POINTER(AjComm)()
        binding._check(binding.lib().aj_comm_nccl_create(ctypes.byref(self.h), path, raw, self.world, self.rank))

    def ptr(self):
        return self.h

    def free(self):
        from . import binding
        if self.h:
            binding._check(binding.lib().aj_comm_nccl_free(self.h))
            self.h = ctypes.POINTER(AjComm)()


def nccl_library_path():
    """The libnccl.so.2 torch ships (so the process holds a single NCCL), else the default."""
    import glob
    import os
    try:
        import nvidia.nccl
        for d in nvidia.nccl.__path__:
            hits = glob.glob(os.path.join(d, "lib", "libnccl.so*"))
            if hits:
                return sorted(hits)[0].encode()
    except Exception:
        pass
    return None
