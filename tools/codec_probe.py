"""Wire codec kernels at the C5 row shape [512, 14336], timed
through the C-ABI with preallocated device buffers (the Python codec API adds
a finiteness check with a host sync, which is not the kernel): blockwise int8
quantize and dequantize, CUDA events, L2 flushed between iterations.
Algorithmic bytes per element: 4 (f32) + 1 (code) + 4/64 (scale).

  python tools/codec_probe.py [--rows 512] [--hidden 14336] [--iters 50]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=512)
    p.add_argument("--hidden", type=int, default=14336)
    p.add_argument("--iters", type=int, default=50)
    a = p.parse_args()
    import torch

    from paper_2209_01188_b200 import _lib

    L = _lib.lib()
    x = torch.randn(a.rows, a.hidden, device="cuda") * 0.05
    n = x.numel()
    codes = torch.empty(n, dtype=torch.int8, device="cuda")
    scales = torch.empty(-(-n // 64), device="cuda")
    y = torch.empty_like(x)
    st = _lib.stream_ptr()
    quant = lambda: _lib.check(L.pb_quantize_blockwise(_lib.ptr(x), n, 64, _lib.ptr(codes), _lib.ptr(scales), st))  # noqa: E731
    dequant = lambda: _lib.check(L.pb_dequantize_blockwise(_lib.ptr(codes), _lib.ptr(scales), n, 64, _lib.ptr(y), st))  # noqa: E731
    quant()
    dequant()
    torch.cuda.synchronize()
    peak = 6459.0
    pk = os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = json.load(open(pk))["hbm_gbs"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2 (126 MB) between iterations
    out = {}
    for name, fn in (("quantize", quant), ("dequantize", dequant)):
        ms = 0.0
        for _ in range(a.iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        ms /= a.iters
        gbs = (5 * n + 4 * (n // 64)) / (ms / 1e3) / 1e9
        out[name] = {"us": 1e3 * ms, "GB/s": gbs, "frac_of_measured_hbm": gbs / peak}
    print(json.dumps({"shape": [a.rows, a.hidden], "l2": "256 MB flush between iterations", **out}))


if __name__ == "__main__":
    main()
