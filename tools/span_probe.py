"""Decode step time of a span of --blocks blocks in isolation (batch-1,
synthetic KV context, int8 wire codes in and out like a pipeline stage):
separates a span step's own cost from pipeline hop costs.

  python tools/span_probe.py --blocks 18 --ctx 2048 --steps 20
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--blocks", type=int, default=18)
    p.add_argument("--ctx", type=int, default=2048)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--codes", type=int, default=1, help="int8 wire codes in/out (pipeline stage)")
    p.add_argument("--batch", type=int, default=1, help="batch-1 sessions per step")
    p.add_argument("--profile", type=int, default=0, help="print per-kind live kernel times")
    args = p.parse_args()
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    B = args.batch
    span = BlockSpan(cfg, 0, args.blocks, int8=True, page_tokens=64, n_pages=B * (args.ctx // 64 + 2) + 2,
                     max_tokens=64, max_seqs=B)
    span.generate_weights(42)
    seqs = [span.new_sequence() for _ in range(B)]
    for seq in seqs:
        span._reserve(seq, args.ctx - args.steps - 8)
        seq.length = args.ctx - args.steps - 8
    d = cfg.hidden
    x = torch.randn(B, d, device="cuda") * 0.05
    codes = torch.zeros(B * d, dtype=torch.int8, device="cuda")
    scales = torch.ones(B * d // 64, device="cuda") * 0.001
    oc = torch.empty(B * d, dtype=torch.int8, device="cuda")
    osc = torch.empty(B * d // 64, device="cuda")
    out = torch.empty(B, d, device="cuda")

    def one():
        if args.codes:
            span.step_codes(seqs, [1] * B, in_codes=codes, in_scales=scales, out_codes=oc, out_scales=osc,
                            out_f32=out)
        else:
            span.step([(sq, x[i:i + 1]) for i, sq in enumerate(seqs)], out=out)

    for _ in range(4):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(f"{args.shape} {args.blocks} blocks, batch {B}: {ms:.3f} ms/step = {ms / args.blocks * 1e3:.1f} us/block "
          f"(codes={args.codes})")
    if args.profile:
        span.profile(True)
        for _ in range(args.steps):
            one()
        torch.cuda.synchronize()
        for name, kind in (("gemv", 0), ("attention", 1), ("prologue", 2), ("codec", 4)):
            kms, n, b = span.profile_read(kind)
            if n:
                print(f"  {name}: {n // args.steps} launches/step, {1e3 * kms / n:.1f} us/launch, "
                      f"{b / max(kms, 1e-9) / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
