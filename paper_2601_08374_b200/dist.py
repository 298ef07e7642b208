"""Host-side plumbing for the z-slab decomposition (P^T of A = P^T G^T B^T D B G P).

The library owns the data path (kernels + NCCL exchange inside elas_apply).  This module
holds the small host logic around it, device-agnostic so that it runs under torch.distributed
with NCCL on B200 and with gloo on CPU in the tests:

* ``slab_planes``: the node-plane range [K0, K1] (both ends) a rank holds;
* ``exchange_partial_planes``: the external-exchange mode's halo swap (isend/irecv of the
  partial interface planes with the z-neighbours) -- its result is what elas_interface_add
  consumes;
* ``gather_global``: assemble the global vector on rank 0 (interface planes are replicated,
  rank r > 0 drops its first plane).
"""

from . import elas


def slab_planes(nz, p, rank, nranks):
    b, e = elas.elas_slab_range(nz, rank, nranks)
    return b * p, e * p


def _planes(y_local, plane):
    return y_local.view(3, -1, plane)


def exchange_partial_planes(y_local, plane, rank, nranks, group=None):
    """Send this rank's partial first/last planes to r-1/r+1 and receive theirs.

    Returns (lo_halo, hi_halo): the partial plane of rank r-1 (for this rank's first plane)
    and of rank r+1 (for its last plane), each (3 * plane,) contiguous, or None at the ends.
    Must be called on the UNSUMMED local result (before any interface add).
    """
    import torch
    import torch.distributed as dist
    v = _planes(y_local, plane)
    reqs, lo, hi = [], None, None
    if rank > 0:
        send_lo = v[:, 0].contiguous().reshape(-1)
        lo = torch.empty_like(send_lo)
        reqs.append(dist.isend(send_lo, rank - 1, group=group))
        reqs.append(dist.irecv(lo, rank - 1, group=group))
    if rank < nranks - 1:
        send_hi = v[:, -1].contiguous().reshape(-1)
        hi = torch.empty_like(send_hi)
        reqs.append(dist.isend(send_hi, rank + 1, group=group))
        reqs.append(dist.irecv(hi, rank + 1, group=group))
    for r in reqs:
        r.wait()
    return lo, hi


def gather_global(y_local, plane, rank, nranks, group=None):
    """Global component-blocked vector on rank 0 (None elsewhere)."""
    import torch
    import torch.distributed as dist
    v = _planes(y_local, plane)
    own = v if rank == 0 else v[:, 1:]
    own = own.contiguous()
    if rank != 0:
        dist.send(torch.tensor([own.shape[1]], dtype=torch.int64, device=own.device), 0, group=group)
        dist.send(own, 0, group=group)
        return None
    parts = [own]
    for r in range(1, nranks):
        n = torch.empty(1, dtype=torch.int64, device=own.device)
        dist.recv(n, r, group=group)
        buf = torch.empty((3, int(n.item()), plane), dtype=own.dtype, device=own.device)
        dist.recv(buf, r, group=group)
        parts.append(buf)
    return torch.cat(parts, dim=1).reshape(-1)
