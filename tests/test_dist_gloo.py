"""Multi-process (gloo, CPU) checks of the z-slab decomposition host logic.

Each rank builds its slab as an independent oracle mesh (the partition comes from the
library's own elas_slab_range), computes the LOCAL partial result, swaps partial interface
planes with paper_2601_08374_b200.dist.exchange_partial_planes, adds them on free rows (the
semantics of the library's plane-add kernel) and rank 0 gathers the global vector with
dist.gather_global.  It must equal the global oracle apply (only summation order differs).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

FACES = 1 | 16 | 32      # x-min plus both z faces (z faces belong to the end ranks only)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    return synth.make_problem("d", 3, 2, 7, 2, 4, perturb=True, lognormal_material=True,
                              faces=FACES, seed=41)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_08374_b200 import dist as D
    P = _problem()
    p = P.p
    Nx, Ny, Nz = P.node_dims
    plane = Nx * Ny
    K0, K1 = D.slab_planes(P.nz, p, rank, world)
    b, e = K0 // p, K1 // p
    lam, mu = P.material_arrays()
    faces = FACES & ~(16 | 32)
    if rank == 0:
        faces |= 16
    if rank == world - 1:
        faces |= 32
    m = oracle.Mesh(P.vertex_array()[b:e + 1], p, P.q, lam[b:e], mu[b:e], faces)
    x_local = P.x_slab(K0, K1)
    y_local = torch.from_numpy(oracle.apply(m, x_local))
    lo, hi = D.exchange_partial_planes(y_local, plane, rank, world)
    Z = torch.from_numpy(oracle.constrained_mask(m)).view(3, -1, plane)
    yv = y_local.view(3, -1, plane)
    if lo is not None:
        free = ~Z[:, 0]
        yv[:, 0][free] += lo.view(3, plane)[free]
    if hi is not None:
        free = ~Z[:, -1]
        yv[:, -1][free] += hi.view(3, plane)[free]
    g = D.gather_global(y_local, plane, rank, world)
    if rank == 0:
        out.put(g.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_decomposition_gloo(world):
    P = _problem()
    lam, mu = P.material_arrays()
    y_ref = oracle.apply(oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces), P.x)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    y = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert y.shape == y_ref.shape
    assert np.linalg.norm(y - y_ref) <= 1e-14 * np.linalg.norm(y_ref)
