"""z-slab sharding of the lattice over torch.distributed ranks (north star:
"the lattice shards naturally into z-slabs ... with one-plane halo exchange";
DESIGN.md sect. 6, row (e)).  Argument marshalling and the halo exchange only:
the stencil runs in the CUDA library (spmv_slab), the exchange is NCCL
point-to-point over NVLink on GPUs (gloo on CPU for the host-side tests).

Layout of a rank's extended vector x_ext: (nz + 2) planes of L*L doubles --
plane 0 = the plane below the slab (global z0 - 1, periodic), planes 1..nz =
the slab, plane nz + 1 = the plane above (global z0 + nz).
"""


def slab_bounds(L, rank, world):
    """(z0, nz) of `rank`: contiguous planes, the first L % world ranks one plane more."""
    if not (1 <= world <= L and 0 <= rank < world):
        raise ValueError("need 1 <= world <= L and 0 <= rank < world")
    base, extra = divmod(L, world)
    nz = base + (1 if rank < extra else 0)
    z0 = rank * base + min(rank, extra)
    return z0, nz


def halo_exchange(x_ext, L, nz, group=None):
    """Fill the two halo planes of x_ext from the neighbouring ranks (periodic in z).
    Rank r sends its first slab plane down (to r-1, their upper halo) and its last
    slab plane up (to r+1, their lower halo)."""
    import torch.distributed as dist
    P = L * L
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        x_ext[:P].copy_(x_ext[nz * P:(nz + 1) * P])
        x_ext[(nz + 1) * P:].copy_(x_ext[P:2 * P])
        return x_ext
    rank = dist.get_rank(group)
    down, up = (rank - 1) % world, (rank + 1) % world
    if group is not None:  # P2POp peers are global ranks; down/up are ranks inside `group`
        down, up = dist.get_global_rank(group, down), dist.get_global_rank(group, up)
    first, last = x_ext[P:2 * P], x_ext[nz * P:(nz + 1) * P]
    lo, hi = x_ext[:P], x_ext[(nz + 1) * P:(nz + 2) * P]
    # posting order matters when down == up (two ranks): messages between a pair are
    # matched in order, so every rank sends (last -> up) before (first -> down) and
    # receives (lower halo <- down) before (upper halo <- up)
    ops = [dist.P2POp(dist.isend, last.contiguous(), up, group), dist.P2POp(dist.isend, first.contiguous(), down, group),
           dist.P2POp(dist.irecv, lo, down, group), dist.P2POp(dist.irecv, hi, up, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    return x_ext


def spmv_sharded(y, x_ext, eps, L, nz, hop, sigma=0.0, group=None):
    """y = (A - sigma I) x on this rank's slab: halo exchange, then the slab stencil kernel."""
    from . import binding
    halo_exchange(x_ext, L, nz, group)
    return binding.spmv_slab(y, x_ext, eps, L, nz, hop, sigma)
