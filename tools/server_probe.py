"""STEP over TCP vs the span step it wraps (SURVEY §8 f3 evidence): a B200
span server hosting --blocks blocks of a named shape (seed weights), driven by
the REFERENCE transport (baseline/_ref swarmlm.transport.rpc_call) with f32
and int8 hidden-state payloads; prints the per-step wall time of the RPC and
of the bare span step, i.e. the host/TCP/codec overhead per hop.

  python tools/server_probe.py --blocks 2 --steps 30
"""

import argparse
import os as _os

_os.environ.setdefault("PB_SERVER_TIMING", "1")
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--blocks", type=int, default=2)
    p.add_argument("--steps", type=int, default=30)
    args = p.parse_args()
    import numpy as np
    import torch
    from swarmlm.transport import ENC_F32, ENC_INT8, MSG, encode_tensor, rpc_call

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.server import ServerConfig, ServerNode

    cfg = SHAPES[args.shape]
    res = {}
    for quant, enc in (("none", ENC_F32), ("both", ENC_INT8)):
        node = ServerNode(ServerConfig(seed=42, model=cfg, blocks=(0, args.blocks), quantize=quant, measure_steps=3,
                                       capacity=4, kv_pages=40)).start()
        try:
            sid = os.urandom(16)
            rpc_call(node.address, MSG.OPEN_SESSION, sid + struct.pack(">I", 512), 5000.0)
            rng = np.random.default_rng(0)
            pos = 0
            h = (rng.standard_normal((16, cfg.hidden)) * 0.05).astype(np.float32)
            rpc_call(node.address, MSG.STEP, sid + struct.pack(">I", pos) + encode_tensor(h, enc), 60000.0)
            pos += 16
            x = (rng.standard_normal((1, cfg.hidden)) * 0.05).astype(np.float32)
            for _ in range(3):
                rpc_call(node.address, MSG.STEP, sid + struct.pack(">I", pos) + encode_tensor(x, enc), 60000.0)
                pos += 1
            payload = encode_tensor(x, enc)  # the client's codec is not part of the hop
            t0 = time.perf_counter()
            for _ in range(args.steps):
                rpc_call(node.address, MSG.STEP, sid + struct.pack(">I", pos) + payload, 60000.0)
                pos += 1
            rpc_ms = (time.perf_counter() - t0) / args.steps * 1e3
            if node.timing:
                tt = node.timing[-args.steps:]
                dec, comp, enc = (sum(x[i] for x in tt) / len(tt) * 1e3 for i in range(3))
                print(f"  server phases (ms): decode {dec:.3f}, scheduler+compute {comp:.3f}, encode {enc:.3f}")
            span = node.span
            seq = span.new_sequence()
            xt = torch.from_numpy(x).cuda()
            for _ in range(3):
                span.step([(seq, xt)])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                span.step([(seq, xt)])
                torch.cuda.synchronize()
            span_ms = (time.perf_counter() - t0) / args.steps * 1e3
            span.release(seq)
            res[quant] = (rpc_ms, span_ms)
            print(f"{args.shape} x{args.blocks} blocks, quantize={quant}: STEP rpc {rpc_ms:.3f} ms, bare span step "
                  f"{span_ms:.3f} ms, host/TCP/codec overhead {rpc_ms - span_ms:.3f} ms per hop", flush=True)
        finally:
            node.stop()


if __name__ == "__main__":
    main()
