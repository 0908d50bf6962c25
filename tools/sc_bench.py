"""Stochastic Collocation throughput on one B200: coupled collocation steps of
config 3 at 1024^2 (100 quadrature nodes per cell) through the C-ABI, device-resident node states.
Prints one JSON line: cell-steps/s, node-steps/s, and the HBM bandwidth of the step counted as the
node states read once and written once (8 * 2 Q m bytes per cell-step).
usage: python tools/sc_bench.py [--nx 1024] [--steps 10] [--warmup 3]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from inputs import configs  # noqa: E402
from paper_1912_09238_b200 import Context  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    cfg = configs.get("cfg3", mesh=dict(nx=args.nx, ny=args.nx))
    g = Context(cfg)
    a, b = g.sc_zeros(), g.sc_zeros()
    g.ipm_sc_init(a)
    for _ in range(args.warmup):
        g.ipm_sc_step(a, b, sync=False)
        a, b = b, a
    st = g.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(args.steps):
        g.ipm_sc_step(a, b, sync=False)
        a, b = b, a
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    cells, Q, m = g.cells, g.Q, g.m
    print(json.dumps({"workload": f"cfg3 {args.nx}^2 Stochastic Collocation (coupled steps)", "cells": cells, "Q": Q,
                      "ms_per_step": ms, "cell_steps_per_s": cells / (ms / 1e3),
                      "node_steps_per_s": cells * Q / (ms / 1e3),
                      "hbm_gbs_node_states_rw": cells * Q * m * 16 / (ms / 1e3) / 1e9}))


if __name__ == "__main__":
    main()
