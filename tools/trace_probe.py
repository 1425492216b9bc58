"""Per-CTA timeline of one decode step (pb_trace_set): for every traced launch
(int8 GEMV, attention, operand writer) the spread of CTA entry, dependency
release, first weight stage and finish, relative to the step's first stamp.
Shows where a block's time goes between kernels (ramp, tail, PDL gaps).

  python tools/trace_probe.py --blocks 3 --ctx 2048
"""

import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

KIND = {0: "gemv", 1: "attn", 2: "frag"}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--blocks", type=int, default=3)
    p.add_argument("--ctx", type=int, default=2048)
    p.add_argument("--batch", type=int, default=1)
    p.add_argument("--steps", type=int, default=2, help="traced steps (the last one is printed)")
    p.add_argument("--sm", action="store_true", help="per-SM GEMV streaming rates: are slow SMs the same every launch?")
    p.add_argument("--attn", action="store_true", help="per-CTA attention durations: which CTAs form the tail")
    args = p.parse_args()
    import numpy as np
    import torch

    from paper_2209_01188_b200 import _lib
    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES[args.shape]
    B = args.batch
    span = BlockSpan(cfg, 0, args.blocks, int8=True, page_tokens=64, n_pages=B * (args.ctx // 64 + 2) + 2,
                     max_tokens=64, max_seqs=B)
    span.generate_weights(42)
    seqs = [span.new_sequence() for _ in range(B)]
    for seq in seqs:
        span._reserve(seq, args.ctx - 16)
        seq.length = args.ctx - 16
    d = cfg.hidden
    codes = torch.zeros(B * d, dtype=torch.int8, device="cuda")
    scales = torch.ones(B * d // 64, device="cuda") * 0.001
    oc = torch.empty(B * d, dtype=torch.int8, device="cuda")
    osc = torch.empty(B * d // 64, device="cuda")
    out = torch.empty(B, d, device="cuda")

    def one():
        span.step_codes(seqs, [1] * B, in_codes=codes, in_scales=scales, out_codes=oc, out_scales=osc, out_f32=out)

    for _ in range(4):
        one()
    torch.cuda.synchronize()
    L = _lib.lib()
    cap = 1 << 22
    buf = torch.zeros(cap, dtype=torch.int64, device="cuda")
    for _ in range(args.steps):
        buf.zero_()
        L.pb_trace_set(C.c_void_p(buf.data_ptr()), cap)
        one()
        torch.cuda.synchronize()
    n = L.pb_trace_meta(None, 0)
    meta = (C.c_int64 * (3 * n))()
    L.pb_trace_meta(meta, n)
    L.pb_trace_set(None, 0)
    t = buf.cpu().numpy().view(np.uint64).astype(np.float64)
    recs = []
    for i in range(n):
        kind, ctas, off = meta[3 * i], meta[3 * i + 1], meta[3 * i + 2]
        recs.append((KIND.get(kind, str(kind)), t[off:off + 16 * ctas].reshape(ctas, 16)))
    base = min(r[:, 0][r[:, 0] > 0].min() for _, r in recs)
    us = lambda v: (v - base) / 1e3  # noqa: E731

    def spread(col):
        col = col[col > 0]
        if col.size == 0:
            return "      -       -       -"
        return f"{us(col.min()):7.1f} {us(np.median(col)):7.1f} {us(col.max()):7.1f}"

    print(f"{args.shape} {args.blocks} blocks, batch {B}, ctx {args.ctx}: one traced decode step (us from first stamp)")
    print("  #  kind  ctas | entry min/med/max      | released min/med/max  | 1st stage min/med/max | "
          "end min/med/max        | busy  gap")
    prev_end = None
    for i, (k, r) in enumerate(recs):
        end = r[:, 3][r[:, 3] > 0]
        emax = us(end.max()) if end.size else float("nan")
        busy = emax - (us(r[:, 0][r[:, 0] > 0].min()))
        gap = "" if prev_end is None else f"{emax - prev_end:6.1f}"
        print(f"{i:3d}  {k:4s} {r.shape[0]:5d} | {spread(r[:, 0])} | {spread(r[:, 1])} | {spread(r[:, 2])} | "
              f"{spread(r[:, 3])} | {busy:6.1f} {gap}")
        prev_end = emax
        if k == "gemv" and (r[:, 8] > 0).any():
            print(f"          gemv: operand resolved {spread(r[:, 10])} | 1st operand stage {spread(r[:, 11])} | "
                  f"MMAs done {spread(r[:, 8])} | epilogue done {spread(r[:, 9])}")
            print(f"          gemv: operand stage 3 written {spread(r[:, 6])} | consumer saw stage 1 {spread(r[:, 12])} "
                  f"2 {spread(r[:, 13])} 3 {spread(r[:, 14])}")
        if k == "frag" and (r[:, 5] > 0).any():
            print(f"          frag summaries loaded {spread(r[:, 7])} | stats (warp 0) {spread(r[:, 2])} | "
                  f"CTA barrier {spread(r[:, 5])} | "
                  f"items written {spread(r[:, 6])}")
    if args.sm:
        sm_rates([r for k, r in recs if k == "gemv"], np)
    if args.attn:
        for k, r in recs:
            if k != "attn":
                continue
            ok = (r[:, 1] > 0) & (r[:, 3] > 0)
            dur = (r[:, 3] - r[:, 1]) / 1e3
            idx = np.where(ok)[0]
            order = idx[np.argsort(-dur[idx])]
            sm = r[:, 4].astype(int)
            # CTAs sharing an SM: how much slower is the slower of a pair?
            pairs = {}
            for c in idx:
                pairs.setdefault(sm[c], []).append(dur[c])
            gaps = [max(v) - min(v) for v in pairs.values() if len(v) == 2]
            cross = idx[r[idx, 8] > 0]  # CTAs with a second segment
            if cross.size:
                rel = lambda col: (r[cross, col] - r[cross, 1]) / 1e3  # noqa: E731
                n1 = lambda col: np.median(rel(col))  # noqa: E731
                print(f"attn: {cross.size} CTAs cross a head boundary; median us after release: seg0 start "
                      f"{n1(5):.1f} data {n1(6):.1f} done {n1(7):.1f} | seg1 start {n1(8):.1f} data {n1(9):.1f} "
                      f"done {n1(10):.1f} | end {n1(3):.1f}; single-segment CTAs end "
                      f"{np.median((r[idx[r[idx, 8] == 0], 3] - r[idx[r[idx, 8] == 0], 1]) / 1e3):.1f}")
            rel0 = lambda col: np.median((r[idx, col] - r[idx, 1]) / 1e3)  # noqa: E731
            print(f"attn: median us after release: first segment start {rel0(5):.2f} first K/V data {rel0(6):.2f} "
                  f"stages done {rel0(11):.2f} merged {rel0(12):.2f} segment done {rel0(7):.2f} end {rel0(3):.2f}")
            print(f"attn: release->end p50 {np.median(dur[idx]):.1f} p90 {np.percentile(dur[idx], 90):.1f} "
                  f"max {dur[idx].max():.1f} us; same-SM pair gap median {np.median(gaps) if gaps else 0:.1f} us; "
                  f"slowest CTAs (index, SM, us): " + ", ".join(f"{c}/{sm[c]}/{dur[c]:.1f}" for c in order[:10]))
    span.close()


def sm_rates(gemvs, np):
    """Per-CTA streaming time (first stage -> end) relative to its launch's
    median, averaged per SM over even and over odd launches: a high
    correlation between the two halves means the slow SMs are systematic."""
    n_sm = int(max(r[:, 4].max() for r in gemvs)) + 1
    halves = [np.zeros(n_sm), np.zeros(n_sm)], [np.zeros(n_sm), np.zeros(n_sm)]
    rel_all = []
    for i, r in enumerate(gemvs):
        ok = (r[:, 2] > 0) & (r[:, 3] > 0)
        dur = r[ok, 3] - r[ok, 2]
        rel = dur / np.median(dur)
        rel_all.append(rel)
        sm = r[ok, 4].astype(int)
        np.add.at(halves[0][i % 2], sm, rel)
        np.add.at(halves[1][i % 2], sm, 1)
    a = halves[0][0] / np.maximum(halves[1][0], 1)
    b = halves[0][1] / np.maximum(halves[1][1], 1)
    m = (halves[1][0] > 0) & (halves[1][1] > 0)
    rel = np.concatenate(rel_all)
    print(f"GEMV launches {len(gemvs)}: per-CTA time / launch median: p5 {np.percentile(rel, 5):.3f} "
          f"p50 1.000 p95 {np.percentile(rel, 95):.3f} max {rel.max():.3f}")
    print(f"per-SM mean (even launches) vs (odd launches): corr {np.corrcoef(a[m], b[m])[0, 1]:.3f}, "
          f"per-SM spread p5 {np.percentile(a[m], 5):.3f} p95 {np.percentile(a[m], 95):.3f}")
    order = np.argsort(-(a + b))
    print("slowest SMs (even, odd):", ", ".join(f"{s}:{a[s]:.3f}/{b[s]:.3f}" for s in order[:8]))
    print("fastest SMs (even, odd):", ", ".join(f"{s}:{a[s]:.3f}/{b[s]:.3f}" for s in order[-8:]))


if __name__ == "__main__":
    main()
