"""Config-2 (BLOOM-560M shape, 24 blocks on one GPU) decode step: host enqueue
time vs device time per step, and the per-kind device split -- is the small
shape bound by the CPU issuing launches or by the GPU's per-kernel latency?

  python tools/c2_probe.py [--steps 50]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--shape", default="bloom-560m")
    p.add_argument("--blocks", type=int, default=0)
    p.add_argument("--no-graphs", action="store_true", help="launch kernel by kernel (no CUDA graph replay)")
    a = p.parse_args()
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[a.shape]
    L = a.blocks or cfg.n_layers
    span = BlockSpan(cfg, 0, L, int8=True, page_tokens=64, n_pages=8, max_tokens=128, max_seqs=2,
                     graphs=not a.no_graphs)
    span.generate_weights(42)
    seq = span.new_sequence()
    g = torch.Generator(device="cuda").manual_seed(3)
    span.step([(seq, torch.randn(128, cfg.hidden, device="cuda", generator=g) * 0.05)])
    x1 = torch.randn(1, cfg.hidden, device="cuda", generator=g) * 0.05
    out = torch.empty_like(x1)
    for _ in range(5):
        span.step([(seq, x1)], out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(a.steps):
        span.step([(seq, x1)], out=out)
    t_issue = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t0
    dev_ms = e0.elapsed_time(e1) / a.steps
    # device-only time: a long queue of steps behind a blocking kernel, so the CPU runs ahead
    print(f"{a.shape} {L} blocks: device {dev_ms * 1e3:.1f} us/step ({dev_ms * 1e3 / L:.1f} us/block), "
          f"host issue {t_issue / a.steps * 1e6:.1f} us/step, wall {t_wall / a.steps * 1e6:.1f} us/step, "
          f"launches/step {span.last_launches}", flush=True)
    span.profile(True)
    for _ in range(5):
        span.step([(seq, x1)], out=out)
    torch.cuda.synchronize()
    kinds = {n: span.profile_read(k) for n, k in (("gemv", 0), ("attn", 1), ("prologue", 2), ("codec", 4))}
    span.profile(False)
    print({n: (round(1e3 * v[0] / 5, 1), v[1] // 5) for n, v in kinds.items() if v[1]}, "(us per step, launches per step)")


if __name__ == "__main__":
    main()
