"""Distributed CUDA path over NCCL (one process per GPU, the bench's multi-GPU launch): 2 ranks own
the halves of a config-3 mesh, exchange boundary duals with NCCL point-to-point and all-reduce the
CFL rate (paper_1912_09238_b200.dist), and the assembled moments must equal a single-GPU run bit for
bit and the oracle to 1e-9 (reading 27).  Needs >= 2 GPUs: skipped on a one-GPU box (the gloo tests
in test_distributed_cpu.py and the virtual ranks of test_gpu_partition.py cover the logic there)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from inputs import configs

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    return configs.get("cfg3", mesh=dict(nx=32, ny=24))


def _worker(rank, world, port, outdir, steps):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    from paper_1912_09238_b200 import Context

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    g = Context(_cfg(), rank=rank, nranks=world, px=2, py=1)
    u = g.zeros()
    g.ipm_project_ic(u)
    lam = g.zeros()
    g.ipm_warm_start(u, lam)
    for _ in range(steps):
        info = g.ipm_step(u, lam, 1e9)
        assert info.failed_cells == 0
    np.save(os.path.join(outdir, f"u{rank}.npy"), u.cpu().numpy())
    np.save(os.path.join(outdir, f"ids{rank}.npy"), g.cell_ids())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_nccl_matches_single_gpu_and_oracle():
    import torch
    import torch.multiprocessing as mp

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (one process per GPU over NCCL)")
    import oracle
    from paper_1912_09238_b200 import Context

    from .gpu_common import assert_moments_close

    steps = 5
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(2, _port(), d, steps), nprocs=2, join=True)
        ref = Context(_cfg())
        u_ref, _, _ = ref.run(n_steps=steps, t_end=1e9)
        ur = u_ref.cpu().numpy()
        out = np.zeros_like(ur)
        for r in range(2):
            ids = np.load(os.path.join(d, f"ids{r}.npy"))
            out[ids] = np.load(os.path.join(d, f"u{r}.npy"))
    np.testing.assert_array_equal(out, ur)
    u_o, _, _ = oracle.Oracle(_cfg()).run(n_steps=steps, t_end=1e9)
    assert_moments_close(out, u_o, 1e-9, "2-rank NCCL")
