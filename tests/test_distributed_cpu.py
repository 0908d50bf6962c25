"""Multi-rank path on CPU (gloo, world sizes 2 and 4): libipm's partition and halo lists
(ipm_partition_query, the same host code ipm_init uses) plus the product's exchange step
(paper_1912_09238_b200.dist over torch.distributed) drive a rank-local oracle; the owned cells must
reproduce a single-process oracle run bit for bit (the dual problems are cell-local, the CFL maximum
is exact, the flux reads only face neighbours: partition invariance)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from inputs import configs
from inputs.generators import bump_channel_mesh


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(name):
    if name == "cart":
        cfg = configs.get("cfg3", mesh=dict(nx=12, ny=10), t_end=None)
        return cfg, None
    if name == "1d":
        cfg = configs.get("cfg2", mesh=dict(nx=60), M=4, q1d=8, t_end=None)
        return cfg, None
    cfg = configs.get("cfg4", mesh=dict(nx_pts=16, ny_pts=7), levels=None, M=3, q1d=6, newton="full",
                      update="conservative")
    m = cfg["mesh"]
    return cfg, bump_channel_mesh(m["nx_pts"], m["ny_pts"], m["seed"])


def _worker(rank, world, port, name, px, py, steps, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1912_09238_b200 import dist as pdist
    from paper_1912_09238_b200 import ipm

    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, ma = _case(name)
    part = ipm.partition_query(cfg, rank, world, px, py, ma)
    o = oracle.Oracle(cfg, ma, n_threads=1)
    u = o.project_ic()
    lam = o.warm_start(u)
    own, send, halo = part["local"], part["send"], part["halo"]
    layout = dict(peers=part["peers"].tolist(), send_count=part["send_count"].tolist(),
                  recv_count=part["recv_count"].tolist())
    row = o.N * o.m
    boundary = np.unique(send)
    interior = np.setdiff1d(own, boundary)
    for _ in range(steps):
        # the binding's order (ipm_step_dual_boundary / _interior): the dual problems of the cells
        # adjacent to a peer first, their duals sent while the interior cells solve (no
        # communication inside the dual problems)
        for j in boundary:
            lam[j], _, _, st = o.dual_solve_cell(u[j], lam[j], cfg["newton"])
            assert st == 0
        sendbuf = torch.from_numpy(np.ascontiguousarray(lam[send].reshape(len(send), row)))
        recvbuf = torch.zeros((len(halo), row), dtype=torch.float64)
        reqs = pdist.halo_exchange(sendbuf, recvbuf, layout, async_op=True)
        for j in interior:
            lam[j], _, _, st = o.dual_solve_cell(u[j], lam[j], cfg["newton"])
            assert st == 0
        pdist.wait_all(reqs)
        lam[halo] = recvbuf.numpy().reshape(len(halo), o.N, o.m)
        rate = np.array([o.cell_rates(lam)[own].max()])
        bits = torch.from_numpy(rate.view(np.int64).copy())
        pdist.allreduce_max_(bits)
        dt = cfg["cfl"] / bits.numpy().view(np.float64)[0]
        new = o.flux_update(lam, u, dt)
        u[own] = new[own]
    np.save(os.path.join(outdir, f"u{rank}.npy"), u[own])
    np.save(os.path.join(outdir, f"ids{rank}.npy"), own)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world,px,py", [("cart", 2, 2, 1), ("cart", 4, 2, 2), ("1d", 2, 0, 0),
                                              ("tri", 2, 0, 0), ("tri", 4, 0, 0)])
def test_partition_invariance_gloo(oracle_mod, name, world, px, py):
    steps = 3
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), name, px, py, steps, d), nprocs=world, join=True)
        cfg, ma = _case(name)
        ref = oracle_mod.Oracle(cfg, ma)
        u_ref, _, _ = ref.run(n_steps=steps)
        seen = np.zeros(ref.cells, bool)
        for r in range(world):
            ids = np.load(os.path.join(d, f"ids{r}.npy"))
            u = np.load(os.path.join(d, f"u{r}.npy"))
            assert not seen[ids].any()
            seen[ids] = True
            np.testing.assert_array_equal(u, u_ref[ids])
        assert seen.all()


def test_partition_lists_are_consistent():
    from paper_1912_09238_b200 import ipm

    for name, world, px, py in [("cart", 4, 2, 2), ("tri", 3, 0, 0), ("1d", 3, 0, 0)]:
        cfg, ma = _case(name)
        parts = [ipm.partition_query(cfg, r, world, px, py, ma) for r in range(world)]
        for r, pr in enumerate(parts):
            s0 = 0
            for peer, ns in zip(pr["peers"], pr["send_count"]):
                mine = pr["send"][s0:s0 + ns]
                other = parts[peer]
                k = list(other["peers"]).index(r)
                r0 = int(np.sum(other["recv_count"][:k]))
                np.testing.assert_array_equal(mine, other["halo"][r0:r0 + other["recv_count"][k]])
                assert set(mine) <= set(pr["local"])
                s0 += ns
