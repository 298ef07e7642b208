"""torchrun worker of tests/test_gpu_multi.py: one process per GPU, NCCL-mode z-slab operators.

Checks the multi-GPU path of the library on real GPUs (A6, PAPER.md:169 P^T):
  1. elas_apply on NCCL slabs (interface planes summed by send/recv overlapped with the interior)
     == the single-GPU apply (<= 1e-14) and == the oracle (<= 1e-12, every row), replicated
     interface planes bitwise equal on both ranks; then the NVLink peer-store exchange
     (elas_set_peer_exchange) bitwise equal to the NCCL one, over several epochs, timed A/B;
  2. the slab dot (elas_dot: owned-dof partials, ncclAllReduce) == the single-GPU dot;
  3. PCG with the slab Chebyshev smoother: iterates after 8 iterations == single GPU (<= 1e-10);
  4. one slab V-cycle (restriction with NCCL interface sums) == the single-GPU V-cycle (<= 1e-10);
  5. config 5 at full size split over the ranks: oracle rows incl. EVERY row of each interface
     plane's sampled set and the single-plane sums (sampled, <= 1e-12).
Rank 0 prints "MULTI OK n=<world size>" when every check passed; any failure raises.
Launch: torchrun --standalone --nproc-per-node N tests/multi_gpu_worker.py [--big]
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist

import oracle
import synth
from paper_2601_08374_b200 import elas
from paper_2601_08374_b200.elas import GMG, Operator


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def gather_slabs(P, y_local, K0, K1, rank, ws):
    """Rank 0 receives every rank's (K0, K1, y slab) and assembles the global vector."""
    parts = [None] * ws if rank == 0 else None
    dist.gather_object((K0, K1, y_local), parts, dst=0)
    if rank != 0:
        return None, None
    Nx, Ny, Nz = P.node_dims
    plane = Nx * Ny
    yg = np.empty((3, Nz, plane))
    for (k0, k1, yl) in parts:
        yg[:, k0:k1 + 1] = yl.reshape(3, -1, plane)
    return yg.reshape(-1), parts


def check_interfaces(parts, plane):
    for (a, b) in zip(parts[:-1], parts[1:]):
        top = a[2].reshape(3, -1, plane)[:, -1]
        bot = b[2].reshape(3, -1, plane)[:, 0]
        assert np.array_equal(top, bot), "replicated interface planes differ"


def main():
    ws = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    lrank = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(lrank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    dev = torch.device("cuda", lrank)

    def new_id():
        obj = [elas.elas_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    # ---- 1. apply --------------------------------------------------------------------------
    p = 6
    P = synth.make_problem("mg", 4, 3, 2 * ws + 1, p, p + 2, perturb=True, lognormal_material=True,
                           faces=1 | 16 | 32, seed=71)
    b, e = elas.elas_slab_range(P.nz, rank, ws)
    K0, K1 = b * p, e * p
    op = Operator.from_problem(P, rank=rank, nranks=ws, nccl_id=new_id())
    xl = torch.from_numpy(P.x_slab(K0, K1)).to(dev)
    yl = torch.empty_like(xl)
    op.apply(xl, yl)
    torch.cuda.synchronize()
    yg, parts = gather_slabs(P, yl.cpu().numpy(), K0, K1, rank, ws)
    if rank == 0:
        Nx, Ny, _ = P.node_dims
        check_interfaces(parts, Nx * Ny)
        one = Operator.from_problem(P)
        x1 = torch.from_numpy(P.x).to(dev)
        y1 = torch.empty_like(x1)
        one.apply(x1, y1)
        torch.cuda.synchronize()
        y1 = y1.cpu().numpy()
        assert rel(yg, y1) <= 1e-14, rel(yg, y1)
        lam, mu = P.material_arrays()
        y_ref = oracle.apply(oracle.Mesh(P.vertex_array(), P.p, P.q, lam, mu, P.dirichlet_faces), P.x)
        assert rel(yg, y_ref) <= 1e-12, rel(yg, y_ref)

    # ---- 1b. NVLink peer-store interface sum: bitwise equal to the NCCL exchange (ws >= 2) ---
    if ws > 1:
        op.set_deterministic(True)               # colored scatter: y bitwise reproducible run to run
        op.apply(xl, yl)
        y_nccl = yl.clone()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        for _ in range(10):
            op.apply(xl, yl)
        ev[1].record()
        op.set_peer_exchange(True)
        yp = torch.empty_like(yl)
        for _ in range(3):                       # several epochs: flags, halo reuse
            op.apply(xl, yp)
            torch.cuda.synchronize()
            assert torch.equal(yp, y_nccl), "peer-store exchange differs from NCCL"
        ev[2].record()
        for _ in range(10):
            op.apply(xl, yp)
        ev[3].record()
        torch.cuda.synchronize()
        assert torch.equal(yp, y_nccl)
        t_nccl, t_peer = ev[0].elapsed_time(ev[1]) / 10, ev[2].elapsed_time(ev[3]) / 10
        times = [None] * ws if rank == 0 else None
        dist.gather_object((t_nccl, t_peer), times, dst=0)
        if rank == 0:
            print(f"apply ms per rank (NCCL exchange, peer store): {times}", flush=True)
        _, parts = gather_slabs(P, yp.cpu().numpy(), K0, K1, rank, ws)
        if rank == 0:
            check_interfaces(parts, P.node_dims[0] * P.node_dims[1])   # replicas bitwise equal
        op.set_peer_exchange(False)
        op.set_deterministic(False)

    # ---- 2. slab dot -------------------------------------------------------------------------
    d = elas.elas_dot(op.h, xl, yl)
    if rank == 0:
        d1 = float(torch.dot(x1, torch.from_numpy(y1).to(dev)))
        assert abs(d - d1) <= 1e-12 * abs(d1), (d, d1)

    # ---- 3. PCG + Chebyshev on NCCL slabs ------------------------------------------------------
    ch = op.chebyshev(order=3, power_iters=10)
    xs = torch.zeros_like(xl)
    op.pcg(xl, xs, precond=elas.PC_CHEBYSHEV, cheb=ch, rtol=0.0, maxit=8)
    torch.cuda.synchronize()
    xsg, parts = gather_slabs(P, xs.cpu().numpy(), K0, K1, rank, ws)
    if rank == 0:
        check_interfaces(parts, Nx * Ny)
        ch1 = one.chebyshev(order=3, power_iters=10)
        x1s = torch.zeros_like(x1)
        one.pcg(x1, x1s, precond=elas.PC_CHEBYSHEV, cheb=ch1, rtol=0.0, maxit=8)
        torch.cuda.synchronize()
        assert rel(xsg, x1s.cpu().numpy()) <= 1e-10, rel(xsg, x1s.cpu().numpy())
        ch1.close()
    ch.close()
    op.close()

    # ---- 4. one V-cycle on NCCL slabs ----------------------------------------------------------
    levels = 2
    Pg = synth.make_problem("mgg", 2, 4, 2 * 2 * ws, 2, 3, perturb=True, lognormal_material=True,
                            faces=1 | 16 | 32, seed=72)
    b, e = elas.elas_slab_range(Pg.nz, rank, ws)
    K0, K1 = b * Pg.p, e * Pg.p
    g = GMG.from_problem(Pg, levels=levels, rank=rank, nranks=ws, nccl_id=new_id())
    rl = torch.from_numpy(Pg.x_slab(K0, K1)).to(dev)
    zl = torch.empty_like(rl)
    g.apply(rl, zl)
    torch.cuda.synchronize()
    zg, parts = gather_slabs(Pg, zl.cpu().numpy(), K0, K1, rank, ws)
    if rank == 0:
        Nx, Ny, _ = Pg.node_dims
        g1 = GMG.from_problem(Pg, levels=levels)
        r1 = torch.from_numpy(Pg.x).to(dev)
        z1 = torch.empty_like(r1)
        g1.apply(r1, z1)
        torch.cuda.synchronize()
        assert rel(zg, z1.cpu().numpy()) <= 1e-10, rel(zg, z1.cpu().numpy())
        g1.close()
    g.close()

    # ---- 5. config 5 at full size, split over the ranks ----------------------------------------
    if "--big" in sys.argv:
        from tests import oracle_pool
        P5 = synth.make_config(5, draw_x=False)
        b, e = elas.elas_slab_range(P5.nz, rank, ws)
        K0, K1 = b * P5.p, e * P5.p
        op5 = Operator.from_problem(P5, rank=rank, nranks=ws, nccl_id=new_id())
        xl = torch.from_numpy(P5.x_slab(K0, K1)).to(dev)
        yl = torch.empty_like(xl)
        op5.apply(xl, yl)
        torch.cuda.synchronize()
        Nx, Ny, Nz = P5.node_dims
        N = Nx * Ny * Nz
        plane = Nx * Ny
        rng = np.random.default_rng(100 + rank)
        # rows of this slab: 1024 random + 256 on each interface plane it holds
        own = [K0 + rng.integers(0, K1 - K0 + 1, 1024)]
        for K in (K0, K1):
            if 0 < K < Nz - 1:
                own.append(np.full(256, K))
        Ks = np.concatenate(own)
        nodes = Ks * plane + rng.integers(0, plane, Ks.size)
        comp = rng.integers(0, 3, Ks.size)
        rows = np.unique(comp * N + nodes)
        local = (rows // N) * (K1 - K0 + 1) * plane + (rows % N - K0 * plane)
        got = yl.cpu().numpy()[local]
        allrows = [None] * ws if rank == 0 else None
        dist.gather_object((rows, got), allrows, dst=0)
        if rank == 0:
            rows = np.concatenate([a for a, _ in allrows])
            got = np.concatenate([b_ for _, b_ in allrows])
            P5x = synth.make_config(5)
            lam, mu = P5x.material_arrays()
            m5 = oracle.Mesh(P5x.vertex_array(), P5x.p, P5x.q, lam, mu, P5x.dirichlet_faces)
            ref = oracle_pool.apply_rows(m5, P5x.x, rows)
            assert rel(got, ref) <= 1e-12, rel(got, ref)
        op5.close()

    dist.barrier()
    if rank == 0:
        print(f"MULTI OK n={ws}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
