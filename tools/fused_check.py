"""Writes the hidden states of a few decode steps (560M shape, 3 blocks, and
176B shape, 1 block with outlier features; batch 1 and 2) to the .npy file
given as argv[1]; run once with argv[2] == "kernel" (operands built by
k_fragwrite, BlockSpan(operand_kernel=True)) and once without (the GEMV's own
operand warps) to compare them (tests/test_gpu_fused.py)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    kernel = len(sys.argv) > 2 and sys.argv[2] == "kernel"
    flat = []
    for name, L, thr, boost in (("bloom-560m", 3, 0.049995, 0.0), ("bloom-176b", 1, 6.0, 200.0)):
        cfg = SHAPES[name]
        span = BlockSpan(cfg, 0, L, int8=True, page_tokens=16, max_tokens=64, max_seqs=2, outlier_threshold=thr,
                         operand_kernel=kernel, n_pages=16)
        span.generate_weights(42, outlier_boost=boost, boost_every=97 if boost else 0)
        g = torch.Generator(device="cuda")
        g.manual_seed(3)
        outs = []
        seqs = [span.new_sequence(), span.new_sequence()]
        x = torch.randn(20, cfg.hidden, generator=g, device="cuda") * 0.5
        outs.append(span.step([(seqs[0], x[:12]), (seqs[1], x[12:20])]))  # prefill (12 + 8 tokens)
        for _ in range(4):
            y = torch.randn(2, cfg.hidden, generator=g, device="cuda") * 0.5
            outs.append(span.step([(seqs[0], y[:1])]))  # 1 token
            outs.append(span.step([(seqs[0], y[:1]), (seqs[1], y[1:])]))  # 2 tokens
        flat += [t.cpu().numpy().reshape(-1) for r in outs for t in r]
        print(name, "outliers per matrix of block 0:", [span.outliers(0, m).size for m in range(4)])
        span.close()
        torch.cuda.empty_cache()
    np.save(sys.argv[1], np.concatenate(flat))

if __name__ == "__main__":
    main()
