#!/usr/bin/env python
"""Feasibility probe (not part of the product): does running GroupNorm applies concurrently with
convs on a partitioned GPU beat running them back to back under the power cap?

Two half-batches (16 images of 128 ch at 1024^2).  Each step of a half = conv3x3 c128 (+residual,
+GN statistics) followed by the GroupNorm+SiLU apply of its output.  'serial': both halves on one
stream with full grids.  'overlap': one stream per half, GEMM grids capped at G SMs and applies at
A SMs (lbx_op_set_grid_limits), so an apply of one half can run beside a conv of the other.
  python scripts/overlap_probe.py --secs 4
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--secs", type=float, default=4.0)
    ap.add_argument("--b", type=int, default=16)
    ap.add_argument("--splits", default="148:148,128:20,120:28,132:16")
    a = ap.parse_args()
    dev = torch.device("cuda")
    b, hw, c = a.b, 1024, 128
    M, K = b * hw * hw, 9 * c
    halves = []
    for _ in range(2):
        x = (torch.randn(b, hw, hw, c, device=dev) * 0.5).half()
        y = torch.empty_like(x)
        w = (torch.randn(c, K, device=dev) * K ** -0.5).half()
        bias = torch.randn(c, device=dev)
        st = lbx.gn_stats_buffer(b)
        gam, bet = torch.ones(c, device=dev), torch.zeros(c, device=dev)
        halves.append((x, y, w, bias, st, gam, bet))
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]

    def step(h, s):
        x, y, w, bias, st, gam, bet = halves[h]
        lbx.op_gemm(1, M, c, K, x.data_ptr(), K, w.data_ptr(), K, y.data_ptr(), c, b=b, h=hw, w=hw, c=c,
                    bias=bias.data_ptr(), resid=x.data_ptr(), ldr=c, gn_stats=st.data_ptr(), stream=s.cuda_stream)
        lbx.op_groupnorm(y.data_ptr(), y.data_ptr(), st.data_ptr(), gam.data_ptr(), bet.data_ptr(), b, hw * hw, c,
                         silu=2, stream=s.cuda_stream)

    def run(mode, gsms, asms):
        lbx.check(lbx.lib().lbx_op_set_grid_limits(gsms, asms))
        torch.cuda.synchronize()
        n, t0 = 0, time.time()
        while time.time() - t0 < a.secs:
            for _ in range(4):
                if mode == "serial":
                    step(0, streams[0]); step(1, streams[0])
                else:
                    step(0, streams[0]); step(1, streams[1])
                n += 1
            torch.cuda.synchronize()
        dt = time.time() - t0
        return dt / n * 1e3  # ms per (both halves) step

    run("serial", 0, 0)  # warm
    for sp in a.splits.split(","):
        g, ap_ = (int(v) for v in sp.split(":"))
        ms_s = run("serial", 0, 0)
        ms_o = run("overlap", g, ap_)
        print(f"gemm {g} SMs / apply {ap_} SMs: serial {ms_s:.2f} ms, overlap {ms_o:.2f} ms per step "
              f"({(ms_s / ms_o - 1) * 100:+.1f}%)", flush=True)
    lbx.check(lbx.lib().lbx_op_set_grid_limits(0, 0))


if __name__ == "__main__":
    main()
