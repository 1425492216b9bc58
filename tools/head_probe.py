"""Client head at a named shape: greedy next-token latency via
the int8 candidate pass (+ exact rescoring) vs the exact f64-accumulated
logits, and the candidates' agreement.

  python tools/head_probe.py --shape bloom-176b --steps 20
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--steps", type=int, default=20)
    args = p.parse_args()
    import torch

    from paper_2209_01188_b200.head import ClientHead
    from paper_2209_01188_b200.model import SHAPES

    cfg = SHAPES[args.shape]
    head = ClientHead(cfg, max_tokens=1)
    head.generate_weights(42)
    g = torch.Generator(device="cuda").manual_seed(1)
    xs = [torch.randn(1, cfg.hidden, device="cuda", generator=g) for _ in range(args.steps)]
    tok = torch.empty(1, dtype=torch.int32, device="cuda")
    for x in xs[:3]:
        head.greedy_device(x, tok)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for x in xs:
        head.greedy_device(x, tok)
    e1.record()
    torch.cuda.synchronize()
    greedy_ms = e0.elapsed_time(e1) / len(xs)
    e0.record()
    for x in xs:
        head.lm_head(x)
    e1.record()
    torch.cuda.synchronize()
    exact_ms = e0.elapsed_time(e1) / len(xs)
    agree = sum(head.greedy(x)[0] == int(head.lm_head(x)[0].argmax()) for x in xs)
    gb_int8 = cfg.vocab * cfg.hidden / 1e9
    print(f"{args.shape} head (V={cfg.vocab}, d={cfg.hidden}): greedy {greedy_ms:.3f} ms/token "
          f"({gb_int8:.2f} GB int8 -> {gb_int8 / greedy_ms:.0f} TB/s-equivalent... {gb_int8 / (greedy_ms / 1e3):.0f} GB/s), "
          f"exact f64 logits {exact_ms:.3f} ms/token ({4 * gb_int8 / (exact_ms / 1e3):.0f} GB/s of f32 rows); "
          f"argmax agreement {agree}/{len(xs)}; device bytes {head.device_bytes / 1e9:.1f} GB")


if __name__ == "__main__":
    main()
