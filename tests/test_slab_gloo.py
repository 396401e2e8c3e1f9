"""Host-side logic of the x-slab decomposition with a real process group:
world_size 2 (and 3) over gloo on the CPU.

Each rank takes its slab from tmg_partition (the library's own partition),
fills its ghost columns by point-to-point halo exchange, applies the
matrix-free node-centric Q4 gather (the algorithm of FineOp / the marching
kernels, restated in numpy as test infrastructure) to its owned columns and
all-reduces the dot product. The gathered result must equal the reference's
assembled matvec and global dot -- i.e. ownership, ghost widths and the
exchange directions are what the GPU kernels assume."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2301_07457_b200 as P

GX = 3  # ghost columns per side (tmg_device.cuh kGX)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def slab_apply(u, E, fixed, ke, ncol, ny):
    """node-centric gather on local columns 0..ncol-1 of a ghosted slab.
    u: [ncol + 2 GX, ny + 1, 2]; E: [ncol + 2 GX, ny] (element column of local
    column c, zero outside the mesh); fixed: same shape as u (bool)."""
    um = np.where(fixed, 0.0, u)
    out = np.zeros((ncol, ny + 1, 2))
    corners = [(0, 0), (1, 0), (1, 1), (0, 1)]  # CCW from lower left (fem.cpp:83-86)
    for sx in (0, 1):
        for sy in (0, 1):
            lx, ly = 1 - sx, 1 - sy  # node's corner inside element (x-1+sx, y-1+sy)
            a = corners.index((lx, ly))
            for b, (cx, cy) in enumerate(corners):
                dx, dy = cx - lx, cy - ly
                for c in range(2):
                    for d in range(2):
                        k = ke[2 * a + c, 2 * b + d]
                        for x in range(ncol):
                            ex = x + GX - lx
                            nbx = x + GX + dx
                            for y in range(ny + 1):
                                ey = y - ly
                                if ey < 0 or ey >= ny:
                                    continue
                                yy = y + dy
                                if yy < 0 or yy > ny:
                                    continue
                                out[x, y, c] += E[ex, ey] * k * um[nbx, yy, d]
    own = fixed[GX:GX + ncol]
    return np.where(own, u[GX:GX + ncol], out)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nc = 32, 8, 2
    rng = np.random.default_rng(5)
    E = rng.uniform(0.05, 1.5, nx * ny)
    ug = rng.standard_normal(2 * (nx + 1) * (ny + 1))
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    x0s, rep = P.slab_partition(nx, ny, nc, world, replicated_level=1)
    x0, x1 = x0s[rank], x0s[rank + 1]
    ncol = x1 - x0
    # owned node data, ghost columns filled by the exchange below
    U = np.zeros((ncol + 2 * GX, ny + 1, 2))
    U[GX:GX + ncol] = ug.reshape(nx + 1, ny + 1, 2)[x0:x1]
    fx = np.zeros(2 * (nx + 1) * (ny + 1), bool)
    fx[bc.fixed_dofs] = True
    FX = np.zeros_like(U, bool)
    Eg = E.reshape(nx, ny)
    EL = np.zeros((ncol + 2 * GX, ny))
    for lx in range(-GX, ncol + GX):
        x = x0 + lx
        if 0 <= x <= nx:
            FX[lx + GX] = fx.reshape(nx + 1, ny + 1, 2)[x]
        if 0 <= x < nx:
            EL[lx + GX] = Eg[x]
    # halo exchange (Comm::halo): my first columns to the left neighbour's
    # right ghost, my last to the right neighbour's left ghost
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(U[GX:GX + 1])), rank - 1))
        left = torch.zeros(GX, ny + 1, 2, dtype=torch.float64)
        reqs.append(dist.irecv(left, rank - 1))
    if rank + 1 < world:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(U[GX + ncol - GX:GX + ncol])), rank + 1))
        right = torch.zeros(1, ny + 1, 2, dtype=torch.float64)
        reqs.append(dist.irecv(right, rank + 1))
    for r in reqs:
        r.wait()
    if rank > 0:
        U[0:GX] = left.numpy()
    if rank + 1 < world:
        U[GX + ncol:GX + ncol + 1] = right.numpy()
    ke = P.element_stiffness(1.0, 0.3)
    Y = slab_apply(U, EL, FX, ke, ncol, ny)
    part = torch.tensor([float(np.sum(U[GX:GX + ncol] * Y))], dtype=torch.float64)
    dist.all_reduce(part)
    pieces = [None] * world
    dist.all_gather_object(pieces, (x0, Y))
    if rank == 0:
        full = np.zeros((nx + 1, ny + 1, 2))
        for a, y in pieces:
            full[a:a + y.shape[0]] = y
        q.put((full.ravel(), part.item(), x0s, rep))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_halo_apply_and_allreduce_over_gloo(world):
    from oracle import pyoracle as po

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    y, dot, x0s, rep = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    nx, ny = 32, 8
    rng = np.random.default_rng(5)
    E = rng.uniform(0.05, 1.5, nx * ny)
    ug = rng.standard_normal(2 * (nx + 1) * (ny + 1))
    g = P.GridLevel(nx, ny)
    bc = P.wall_boundary_conditions(g, "uniform")
    s = po.System("orc", nx, ny, E, 0.3, bc.fixed_dofs, bc.point_loads)
    want = s.matvec(0, ug)
    assert np.max(np.abs(y - want)) <= 1e-13 * np.max(np.abs(want))
    assert abs(dot - float(ug @ want)) <= 1e-12 * abs(float(ug @ want))
    assert len(x0s) == world + 1 and rep == 1


def red_tx(nx, ny):
    """Reduction tile width (tmg_gpu.cu red_tx_of / pow2_strip): the power of
    two in [1, 64] minimising waves x (tx + 3) for 3 x 148 resident CTAs."""
    rows_tiles, cols, slots = -(-(ny + 1) // 128), nx + 1, 3 * 148
    best, best_cost = 64, None
    for tx in (64, 32, 16, 8, 4, 2, 1):
        cost = -(-rows_tiles * -(-cols // tx) // slots) * (tx + 3)
        if best_cost is None or cost < best_cost:
            best, best_cost = tx, cost
    return best


def test_partition_invariants():
    for nx, ny, nc, n in [(8192, 8192, 10, 8), (2048, 2048, 8, 4), (512, 512, 6, 2), (128, 64, 4, 3)]:
        x0s, rep = P.slab_partition(nx, ny, nc, n)
        gran = max(1 << (nc - rep), red_tx(nx, ny))
        assert x0s[0] == 0 and x0s[-1] == nx + 1
        # slab boundaries never split a reduction tile or a coarse column pair
        assert all(x % gran == 0 for x in x0s[:-1])
        assert all(b - a >= 2 * gran for a, b in zip(x0s, x0s[1:]))
    assert red_tx(8192, 8192) == 64 and red_tx(512, 512) == 8 and red_tx(64, 64) == 1
    # one rank keeps every level global
    assert P.slab_partition(64, 64, 3, 1) == ([0, 65], 3)
