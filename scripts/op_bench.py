#!/usr/bin/env python
"""Run single kernels of the path through the C ABI at realistic sizes (for ncu captures and
per-op timing).  Not part of the product; device buffers come from torch (plumbing only).

  python scripts/op_bench.py conv --b 4 --hw 1024 --c 128 --n 128 --resid --stats
  python scripts/op_bench.py subpix --b 4 --hw 512 --c 256
  python scripts/op_bench.py gn --b 4 --hw 1024 --c 128
  python scripts/op_bench.py tail --b 32 --hw 1024      # GroupNorm+SiLU+conv_out+u8 (GB/s of 256 B/px in + 3 out)
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19385_b200 as lbx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("op", choices=["conv", "subpix", "gemm", "gn", "tail"])
    ap.add_argument("--b", type=int, default=4)
    ap.add_argument("--hw", type=int, default=1024)
    ap.add_argument("--c", type=int, default=128)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--resid", action="store_true")
    ap.add_argument("--fold", action="store_true", help="residual as an extra K segment (identity B)")
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--gnfuse", action="store_true", help="fused GroupNorm+SiLU on the A operand")
    ap.add_argument("--inplace", action="store_true", help="gn: apply in place")
    ap.add_argument("--nobias", action="store_true")
    ap.add_argument("--cg", type=int, default=0)
    ap.add_argument("--bn", type=int, default=0)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--bits", type=int, default=1, help="lbx_op_set_debug halo_policy bits")
    ap.add_argument("--sustain", type=float, default=0.0,
                    help="run back to back for this many seconds under nvidia-smi sampling (power-capped rate, J/unit)")
    a = ap.parse_args()
    lbx.check(lbx.lib().lbx_op_set_debug(a.bits, 0))
    dev = torch.device("cuda")
    b, hw, c = a.b, a.hw, a.c
    n = a.n or c
    x = (torch.randn(b, hw, hw, c, device=dev) * 0.5).half()
    stats = lbx.gn_stats_buffer(b)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    if a.op in ("conv", "subpix", "gemm"):
        if a.op == "conv":
            K = 9 * c
            w = (torch.randn(n, K + (n if a.fold else 0), device=dev) * K ** -0.5).half()
            out = torch.empty(b, hw, hw, n, dtype=torch.half, device=dev)
            M, mode, flops = b * hw * hw, 1, 2.0 * b * hw * hw * n * K
        elif a.op == "subpix":
            K = 4 * c
            w = (torch.randn(4 * n, K, device=dev) * K ** -0.5).half()
            out = torch.empty(b, 2 * hw, 2 * hw, n, dtype=torch.half, device=dev)
            M, mode, flops = b * hw * hw, 2, 2.0 * 4 * b * hw * hw * n * 9 * c
        else:
            K = a.k or c
            w = (torch.randn(n, K, device=dev) * K ** -0.5).half()
            x = (torch.randn(b * hw * hw, K, device=dev)).half()
            out = torch.empty(b * hw * hw, n, dtype=torch.half, device=dev)
            M, mode, flops = b * hw * hw, 0, 2.0 * b * hw * hw * n * K
        bias = torch.randn(n, device=dev)
        resid = torch.randn_like(out) if a.resid else None

        fold = a.fold and a.op == "conv"
        gss = (torch.rand(b, c, 2, device=dev) + 0.5) if a.gnfuse else None
        xr = torch.randn_like(out) if fold else None

        def run():
            stats.zero_()
            lbx.op_gemm(mode, M, n, K, x.data_ptr(), K, w.data_ptr(), K + (n if fold else 0), out.data_ptr(), n,
                        b=b, h=hw, w=hw, c=c, a2=xr.data_ptr() if fold else 0, lda2=n, k2=n if fold else 0,
                        bias=0 if a.nobias else bias.data_ptr(), resid=resid.data_ptr() if resid is not None else 0, ldr=n,
                        gn_stats=stats.data_ptr() if a.stats else 0, cta_group=a.cg, bn=a.bn,
                        gn_ss=gss.data_ptr() if gss is not None else 0)
    elif a.op == "tail":
        c = 128
        x = (torch.randn(b, hw, hw, c, device=dev) * 0.5).half()
        ss = torch.stack([torch.rand(b, c, device=dev) + 0.5, torch.randn(b, c, device=dev) * 0.5], dim=-1).contiguous()
        wt = torch.randn(3, 3, 3, c, device=dev) * (9 * c) ** -0.5
        bt = torch.randn(3, device=dev) * 0.2
        rgb = torch.empty(b, hw, hw, 3, dtype=torch.uint8, device=dev)
        flops = float(b * hw * hw * (2 * c + 3))  # bytes

        def run():
            lbx.op_conv_out(x.data_ptr(), ss.data_ptr(), wt.data_ptr(), bt.data_ptr(), rgb.data_ptr(), b, hw, hw,
                            impl=2)
    else:
        gamma = torch.ones(c, device=dev)
        beta = torch.zeros(c, device=dev)
        y = torch.empty_like(x)
        lbx.op_gn_stats(x.data_ptr(), stats.data_ptr(), b, hw * hw, c)
        flops = 4.0 * x.numel()  # bytes
        if a.inplace:
            y = x

        def run():
            lbx.op_groupnorm(x.data_ptr(), y.data_ptr(), stats.data_ptr(), gamma.data_ptr(), beta.data_ptr(), b,
                             hw * hw, c, 2)

    run()
    torch.cuda.synchronize()
    if a.sustain > 0:
        import subprocess
        import time
        unit_scale = 1e9 if a.op in ("gn", "tail") else 1e12
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits",
                                "-lms", "100"], stdout=subprocess.PIPE, text=True)
        t0 = time.time()
        reps = 0
        ev0.record()
        while time.time() - t0 < a.sustain:
            for _ in range(4):
                run()
            reps += 4
            torch.cuda.synchronize()
        ev1.record()
        torch.cuda.synchronize()
        smi.terminate()
        out = smi.communicate()[0].strip().splitlines()
        samples = [tuple(float(v) for v in l.split(",")) for l in out if l.strip()]
        half = samples[len(samples) // 3:]  # skip the ramp
        pw = sum(x[0] for x in half) / max(1, len(half))
        clk = sorted(x[1] for x in half)[len(half) // 2] if half else 0
        ms = ev0.elapsed_time(ev1) / reps
        rate = flops / (ms / 1e3) / unit_scale
        unit = "GB/s" if a.op in ("gn", "tail") else "TFLOP/s(algo)"
        print(f"SUSTAINED {a.op} b{b} hw{hw} c{c} n{n}: {ms:.3f} ms  {rate:.1f} {unit}  power {pw:.0f} W  sm {clk:.0f} MHz  "
              f"{pw / rate:.3f} W per {unit}")
        return
    ev0.record()
    for _ in range(a.iters):
        run()
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / a.iters
    unit = "GB/s" if a.op in ("gn", "tail") else "TFLOP/s(algo)"
    scale = 1e9 if a.op in ("gn", "tail") else 1e12
    print(f"{a.op} b{b} hw{hw} c{c} n{n}: {ms:.3f} ms  {flops / (ms / 1e3) / scale:.1f} {unit}")


if __name__ == "__main__":
    main()
