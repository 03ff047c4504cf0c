"""Kernel micro-benchmarks on the GPU box (development aid, not the bench contract).

    python tools/kbench.py qr        # K4 thin QR at every config's (I_n, K_n)

Times are device times per launch from libtrg's per-kernel CUDA events.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def bench_qr(iters=50):
    import paper_1901_01652_b200 as trg

    ctx = trg.default_context()
    for m, k in [(100, 10), (100, 16), (1000, 20), (1024, 64), (200, 32), (60, 12)]:
        y = np.random.default_rng(0).standard_normal((m, k))
        trg.economy_q(y)
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(iters):
            trg.economy_q(y)
        ctx.set_profiling(False)
        tot, n = ctx.kernel_stats("qr")
        print(f"qr m={m:5d} k={k:3d}: {1e3 * tot / n:8.1f} us/launch")


if __name__ == "__main__" and sys.argv[1] == "qr":
    bench_qr()


def bench_launch_gap(n=200):
    """Back-to-back dependent tiny kernels on one stream: device time per launch."""
    import torch

    x = torch.zeros(1, device="cuda")
    for _ in range(10):
        x.add_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        x.add_(1)
    e1.record()
    torch.cuda.synchronize()
    print(f"launch gap: {1e3 * e0.elapsed_time(e1) / n:.2f} us per dependent tiny kernel")


if __name__ == "__main__" and sys.argv[1] == "gap":
    bench_launch_gap()
