"""Writes the hidden states of a few decode steps (560M shape, 3 blocks,
batch 1 and 2) to the .npy file given as argv[1]; run once with
PB_NO_FUSED_OPERAND=1 and once without to compare the fused-operand GEMV
with the k_fragwrite path (tests/test_gpu_fused.py)."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES["bloom-560m"]
    span = BlockSpan(cfg, 0, 3, int8=True, page_tokens=16, max_tokens=64, max_seqs=2, outlier_threshold=0.049995)
    span.generate_weights(42)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    outs = []
    seqs = [span.new_sequence(), span.new_sequence()]
    x = torch.randn(20, cfg.hidden, generator=g, device="cuda")
    outs.append(span.step([(seqs[0], x[:12]), (seqs[1], x[12:20])]))  # prefill (12 + 8 tokens)
    for _ in range(4):
        y = torch.randn(2, cfg.hidden, generator=g, device="cuda")
        outs.append(span.step([(seqs[0], y[:1])]))  # 1 token
        outs.append(span.step([(seqs[0], y[:1]), (seqs[1], y[1:])]))  # 2 tokens
    np.save(sys.argv[1], np.concatenate([o.cpu().numpy().reshape(-1) for o in [t for r in outs for t in r]]))
    print("outliers per matrix of block 0:", [span.outliers(0, m).size for m in range(4)])


if __name__ == "__main__":
    main()
