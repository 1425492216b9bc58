"""Batched-decode step time per block, IMMA GEMV vs the stream-K tcgen05
kernel (k_gemm_tc_sk), over batch sizes, with synthetic KV context.

  python tools/batch_probe.py --shape bloom-176b --blocks 4 --ctx 64 --batches 1,2,4,8,16,32
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--blocks", type=int, default=4)
    p.add_argument("--ctx", type=int, default=64)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--batches", default="1,2,4,8,16,32")
    p.add_argument("--paths", default="gemv,tc", help="gemv (tc_min_tokens huge) and/or tc (default threshold)")
    p.add_argument("--tc-min", type=int, default=0, help="tc path: tokens from which tcgen05 runs (0: default)")
    args = p.parse_args()
    import json

    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6459.0
    h, L = cfg.hidden, args.blocks
    batches = [int(b) for b in args.batches.split(",")]
    Bmax = max(batches)
    for path in args.paths.split(","):
        span = BlockSpan(cfg, 0, L, int8=True, page_tokens=64, n_pages=Bmax * (args.ctx // 64 + 2) + 2,
                         max_tokens=64, max_seqs=64, tc_min_tokens=100000 if path == "gemv" else args.tc_min)
        span.generate_weights(42)
        for B in batches:
            seqs = [span.new_sequence() for _ in range(B)]
            T = args.ctx - args.steps - 8
            for seq in seqs:
                span.reserve(seq, T)
                seq.length = T
            x = torch.randn(B, h, device="cuda") * 0.05
            out = torch.empty(B, h, device="cuda")

            def one():
                span.step([(sq, x[i:i + 1]) for i, sq in enumerate(seqs)], out=out)

            for _ in range(3):
                one()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                one()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            span.profile(True)
            one()
            torch.cuda.synchronize()
            kinds = {n: span.profile_read(k) for n, k in (("gemv", 0), ("attn", 1), ("prologue", 2), ("tc_sk", 6),
                                                            ("tc", 5))}
            span.profile(False)
            ctx = T + args.steps // 2
            wbytes = L * (12 * h * h + 7 * h * 4 + 13 * h * 4)
            kv = B * L * 2 * ctx * h * 2
            frac = (wbytes + kv) / (peak * 1e9) / (ms / 1e3)
            mm = {n: round(1e3 * v[0], 1) for n, v in kinds.items() if v[1]}
            mat = kinds["tc_sk"] if kinds["tc_sk"][1] else kinds["gemv"]
            mat_gbs = mat[2] / (mat[0] / 1e3) / 1e9 if mat[1] else 0.0
            print(f"{args.shape} {path:4s} B={B:2d}: {1e3 * ms / L:7.1f} us/block  {B / (ms / 1e3):8.1f} tok/s "
                  f"(this span)  HBM frac {frac:.3f}  matmul {mat_gbs:6.0f} GB/s  per-kind us/step {mm}", flush=True)
            for sq in seqs:
                span.release(sq)
        span.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
