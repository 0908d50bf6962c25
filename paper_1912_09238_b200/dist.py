"""The exchange step of the distributed path: torch.distributed plumbing only.

Per (pseudo-)time step, after every rank has solved the dual problems of its own cells:
  * halo_exchange: each rank sends the duals of its cells adjacent to a peer and receives the duals
    of that peer's adjacent cells (one layer of face neighbours: the kinetic flux is a
    nearest-neighbour stencil); NCCL P2P over NVLink on GPUs, gloo on CPU tests.
  * allreduce_max_: the CFL rate (bits of a non-negative double, order-preserving as int64).
  * reduce_info_: step statistics (sums; worst status max) for ipm_step_info.
Buffers are laid out by libipm (ipm_halo_layout): rows [nsend][N*m] / [nrecv][N*m], grouped by
peer in ascending rank order.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _staged(t: torch.Tensor, group) -> bool:
    """gloo has no point-to-point for device tensors: stage through host memory (functional tests of
    the multi-rank path on one GPU; the production backend is NCCL)"""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def halo_exchange(sendbuf: torch.Tensor, recvbuf: torch.Tensor, layout: dict, group=None, async_op=False):
    """async_op: return the requests (wait_all) so that device work queued after this call — the
    interior dual solves — overlaps the transfer; NCCL orders the sends after the work already queued
    on the current stream (the boundary solves and the pack)"""
    if _staged(sendbuf, group):
        rh = recvbuf.cpu()
        halo_exchange(sendbuf.cpu(), rh, layout, group)
        recvbuf.copy_(rh)
        return []
    ops = []
    s0 = r0 = 0
    for peer, ns, nr in zip(layout["peers"], layout["send_count"], layout["recv_count"]):
        if ns:
            ops.append(dist.P2POp(dist.isend, sendbuf[s0:s0 + ns], peer, group))
        if nr:
            ops.append(dist.P2POp(dist.irecv, recvbuf[r0:r0 + nr], peer, group))
        s0 += ns
        r0 += nr
    reqs = dist.batch_isend_irecv(ops) if ops else []
    if async_op:
        return reqs
    wait_all(reqs)
    return []


def wait_all(reqs) -> None:
    for req in reqs:
        req.wait()


def allreduce_max_(t: torch.Tensor, group=None) -> None:
    if _staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        t.copy_(h)
        return
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)


def reduce_info_(info, device, group=None) -> None:
    """Global step statistics from the local ones (ctypes ipm_step_info, in place)."""
    dev = "cpu" if dist.get_backend(group) == "gloo" else device
    nh = len(info.newton_hist)
    v = torch.tensor([info.residual, float(info.newton_iters), float(info.failed_cells), float(info.halvings),
                      float(info.inadmissible_trials)] + [float(x) for x in info.newton_hist],
                     dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    w = torch.tensor([info.worst_status], dtype=torch.int64, device=dev)
    dist.all_reduce(w, op=dist.ReduceOp.MAX, group=group)
    info.residual = float(v[0])
    info.newton_iters = int(v[1])
    info.failed_cells = int(v[2])
    info.halvings = int(v[3])
    info.inadmissible_trials = int(v[4])
    for i in range(nh):
        info.newton_hist[i] = int(v[5 + i])
    info.worst_status = int(w[0])
