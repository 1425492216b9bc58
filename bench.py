"""Headline benchmark: BLOOM-176B-shape int8 decode steps/s (b=1) and tokens/s
(b=32), as a fraction of the HBM roofline (BASELINE.json).

Workload (N GPUs, one process per GPU): the 70-block 176B-shape model
(h=14336, H=112, int8 weights generated on device from the reference's
SplitMix64 streams) is split into N contiguous block spans, one per GPU
(N=1: all 70 blocks on one B200). N batch-1 sessions are in flight (one per
pipeline stage, "weak" scaling: per-GPU work is constant), each decoding at a
context that ends at --ctx (default 2048). A step is one decode token of one
session through all 70 blocks; span-to-span hops carry the hidden state as the
reference's blockwise int8 wire codec through peer-memory mailboxes over
NVLink (pb_hop.cu; `--hop nccl` for NCCL send/recv); the last span hands the
result back to span 0, closing the ring for the session's next token.

value = session-steps/s over all GPUs, CUDA events between barriers, max over
ranks (inputs resident in HBM). Sub-records on the same line:
  e2e    the same metric through the server's public API: client sessions (threads
         of a separate client process) send
         STEP frames (int8 TensorMsg, host bytes) over TCP to the span server
         (N=1: ServerNode; N>1: the box front end, ONE server for [0, 70)
         whose hops stay on the GPUs) and read the replies;
  b32    tokens/s with 32 batch-1 sessions per micro-batch (BASELINE's b=32);
  c2     BLOOM-560M shape on one GPU, 128-token prefix, batch 1 (config 2);
  forward  C5-style FORWARD rows of 512 tokens through the pipeline;
  prefill  the sessions' prompt prefill (480-token tcgen05 jobs);
  f2     BACKWARD of one 512-position row through two 176B blocks;
  cpu_baseline  the reference's arithmetic (oracle port) on the host cores at
         the same context, one block, extrapolated.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "{model} int8 decode steps/s (b=1)"
METRIC_B = "{model} int8 decode tokens/s (b={b})"
RING_BYTES = 64
UNIT = "steps/s"


def model_label(shape: str) -> str:
    return shape.upper()  # bloom-176b -> BLOOM-176B


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--shape", default="bloom-176b")
    p.add_argument("--ctx", type=int, default=2048)
    p.add_argument("--seed", type=int, default=42)
    # a multiple of the tcgen05 GEMM's 80-token tile (256 padded 4 tiles to 320 tokens)
    # tokens per prefill job, a multiple of the 80-token tcgen05 tile (480: prefill 1636 -> 1789 tokens/s and
    # 704 -> 763 useful TFLOP/s against 240; 960 no better)
    p.add_argument("--prefill-chunk", type=int, default=480)
    p.add_argument("--batch", type=int, default=1, help="batch-1 sessions per pipeline micro-batch (headline)")
    p.add_argument("--hop", default="p2p", choices=["p2p", "nccl"],
                   help="span-to-span hop: NVLink peer-memory mailboxes (pb_hop.cu) or NCCL send/recv")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-b32", action="store_true")
    p.add_argument("--no-c2", action="store_true")
    p.add_argument("--no-f2", action="store_true", help="skip the BACKWARD (f2) sub-record")
    p.add_argument("--b32-ctx", type=int, default=64,
                   help="context of the b=32 sessions (N=1: 172.7 GB of weights leave ~8 GB of HBM for KV)")
    p.add_argument("--synthetic-kv", action="store_true", help="skip the real prefill (KV content is synthetic)")
    p.add_argument("--forward-rows", type=int, default=4, help="C5 rows of 512 tokens per GPU")
    return p.parse_args()


# ------------------------------------------------------------------ helpers


from paper_2209_01188_b200.pipeline import split_blocks  # noqa: E402


def bytes_per_step(cfg, ctx_tokens_per_session, n_layers=None):
    """sum_blocks [12h^2 codes + 7h*4 scales + 13h*4 bias/LN]
    + sum_sessions sum_blocks 2*T*h*2 (fp16 K+V)."""
    h, L = cfg.hidden, n_layers or cfg.n_layers
    w = L * (12 * h * h + 7 * h * 4 + 13 * h * 4)
    kv = sum(L * 2 * T * h * 2 for T in ctx_tokens_per_session)
    return w, kv


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([v.strip() for v in out.stdout.strip().split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.1)

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def measured_tflops():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:  # noqa: BLE001
        return 1590.0


def committed_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


# ------------------------------------------------------------------ CPU legs (oracle port)


def cpu_info():
    """CPU model, cores, numpy / BLAS build and thread count."""
    import numpy as np

    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info

        blas = [{k: i.get(k) for k in ("internal_api", "version", "num_threads", "threading_layer")}
                for i in threadpool_info() if i.get("user_api") == "blas"]
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def cpu_block_sample(cfg, ctx):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_baseline

    return cpu_baseline.BlockSample(cfg.hidden, cfg.n_heads, ctx, cfg.mlp_ratio), cpu_baseline.cores()


def cpu_step_seconds(sample, reps, threads=None):
    """Best of `reps` timed samples (OpenBLAS timings are noisy), optionally
    with the BLAS pool limited to `threads`."""
    if threads is None:
        return min(sample.step_seconds() for _ in range(reps))
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=threads, user_api="blas"):
        return min(sample.step_seconds() for _ in range(reps))


def run_reference(args):
    """--impl reference: the reference's CPU arithmetic for one decode step at
    the SAME context (oracle port of block_forward(qw) / matmul_mixed, full
    f32 KV cache concat as model.py:137-151 does), on all host cores; rank 0
    only. A step is a bounded sample: ONE block, timed; value = 1 / (70 x the
    sample time). ms_per_step is the measured sample time, so steps x
    ms_per_step is the timed region."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2209_01188_b200.model import SHAPES

    cfg = SHAPES[args.shape]
    ctx = args.ctx
    sample, ncores = cpu_block_sample(cfg, ctx)
    for _ in range(args.warmup):
        sample.step_seconds()
    ts = [sample.step_seconds() for _ in range(args.steps)]
    per_block = statistics.median(ts)
    value = 1.0 / (per_block * cfg.n_layers)
    desc = (f"1 block of the {args.shape} shape per step, int8-weights decode t=1 at context {ctx} (oracle port of "
            f"quant.py matmul_mixed + model.py block_forward with its f32 KV concat), median of {args.steps}; "
            f"value = 1 / ({cfg.n_layers} x block time)")
    line = {
        "impl": "reference", "metric": METRIC.format(model=model_label(args.shape)), "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_block * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{args.shape} int8 decode b=1 (CPU reference arithmetic)",
                                        "ctx": ctx, "sample": "one block per step, extrapolated x70"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port", "sample": desc,
                         **cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU pipeline


class Pipeline:
    """One span of the model per GPU; jobs follow the deadlock-free ring
    schedule of paper_2209_01188_b200.pipeline. Job ids increase across
    phases (the mailbox flags are monotonic); each phase is its own
    RingSchedule [first, end)."""

    def __init__(self, args, cfg):
        import torch
        import torch.distributed as dist

        from paper_2209_01188_b200.span import BlockSpan

        self.args, self.cfg = args, cfg
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            import datetime

            dist.init_process_group("nccl", device_id=self.dev, timeout=datetime.timedelta(seconds=300))
        self.dist = dist if self.world > 1 else None
        self.S = self.world  # micro-batches in flight (one per pipeline stage)
        self.B = args.batch  # batch-1 sessions per micro-batch
        self.chunk = args.prefill_chunk  # tokens per prefill job (all sessions of the micro-batch)
        self.ranges = split_blocks(cfg.n_layers, self.world)
        s, e = self.ranges[self.rank]
        pages_per_seq = -(-min(cfg.max_seq, args.ctx + 64) // 64)  # KV pool sized for the benchmarked context
        t0 = time.perf_counter()
        self.span = BlockSpan(cfg, s, e, int8=True, page_tokens=64, n_pages=self.S * self.B * pages_per_seq + 2,
                              max_tokens=max(self.chunk, 512), max_seqs=64, device=self.local)
        self.span.generate_weights(args.seed)
        torch.cuda.synchronize()
        self.gen_s = time.perf_counter() - t0
        self.set_batch(self.B)
        d = cfg.hidden
        self.d = d
        cap = self.payload_bytes(max(self.chunk, 512), 1)
        self.inbox = torch.empty(cap, dtype=torch.uint8, device=self.dev)
        self.outbox = torch.empty(cap, dtype=torch.uint8, device=self.dev)
        self.out = torch.empty(max(self.chunk, 512), d, dtype=torch.float32, device=self.dev)
        g = torch.Generator(device=self.dev)
        g.manual_seed(7)
        self.inputs = torch.randn(64, d, generator=g, device=self.dev) * 0.05  # embedding-like rows
        self.launches = 0
        self.next_job = 0
        self.ring = None
        if self.world > 1 and args.hop == "p2p":
            from paper_2209_01188_b200.pipeline import P2PRing

            ok = 1
            try:
                self.ring = P2PRing(self.rank, self.world, self.S, cap, self.local, dist)
            except Exception as e:  # e.g. no CUDA IPC between the processes: every rank falls back together
                print(f"[rank {self.rank}] peer-memory hop unavailable ({e}); using NCCL send/recv", file=sys.stderr)
                ok = 0
            flag = torch.tensor([ok], device=self.dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if not int(flag.item()) and self.ring is not None:
                self.ring.close()
                self.ring = None

    def set_batch(self, B):
        """B batch-1 sessions per micro-batch (fresh sequences; the old ones' pages go back)."""
        for grp in getattr(self, "seqs", []):
            for s in grp:
                self.span.release(s)
        self.B = B
        self.seqs = [[self.span.new_sequence() for _ in range(B)] for _ in range(self.S)]

    def payload_bytes(self, t, B=None):
        n = t * (B or self.B) * self.d
        return -(-n // 16) * 16 + 4 * (-(-n // 64))

    def views(self, buf, t):
        import torch

        n = t * self.B * self.d
        off = -(-n // 16) * 16
        return buf[:n].view(torch.int8), buf[off:off + 4 * (-(-n // 64))].view(torch.float32)

    def barrier(self):
        import torch

        torch.cuda.synchronize()
        if self.dist:
            self.dist.barrier()
        torch.cuda.synchronize()

    def phase(self, lens, fresh=False):
        """One phase: for each entry t of `lens`, one job per micro-batch (S
        jobs), t new positions per session. fresh: release the micro-batch's
        sequences after each job (cache-less FORWARD rows)."""
        first = self.next_job
        jobs = [(first + i * self.S + m, t) for i, t in enumerate(lens) for m in range(self.S)]
        self.next_job = first + len(jobs)
        self.run(jobs, first, self.next_job, fresh=fresh)

    def _input(self, j, n):
        import torch

        if n <= 64:
            return self.inputs[j % 64: j % 64 + 1].expand(n, self.d).contiguous() if n == 1 else self.inputs[:n]
        g = torch.Generator(device=self.dev)
        g.manual_seed(j)
        return torch.randn(n, self.d, device=self.dev, generator=g) * 0.05

    def run(self, jobs, first, end, fresh=False):
        import torch

        from paper_2209_01188_b200.pipeline import RingSchedule, run_jobs, torch_exchange

        sched = RingSchedule(self.rank, self.world, self.S, end, first)
        if self.ring is not None:
            return self.run_p2p(sched, jobs, fresh)
        tmap = dict(jobs)
        r, N = self.rank, self.world

        def step(j, inbox):
            t = tmap[j]
            n = t * self.B
            seqs = self.seqs[j % self.S]
            oc, os_ = self.views(self.outbox, t)
            if inbox is None or r == 0:  # span 0: fresh input (a received ring payload only orders the step)
                self.span.step_codes(seqs, [t] * self.B, in_f32=self._input(j, n), out_codes=oc, out_scales=os_,
                                     out_f32=self.out[:n])
            else:
                ic, is_ = self.views(inbox, t)
                self.span.step_codes(seqs, [t] * self.B, in_codes=ic, in_scales=is_, out_codes=oc, out_scales=os_,
                                     out_f32=self.out[:n])
            self.launches += self.span.last_launches
            if fresh:
                for s in seqs:
                    self.span.release(s)
            if r == N - 1:
                # ring back-edge: only orders span 0's next step of this session
                # (stand-in for the client's LM head); fixed size
                return self.outbox[:RING_BYTES]
            return self.outbox[:self.payload_bytes(t)]

        run_jobs(sched, [j for j, _ in jobs], step, torch_exchange,
                 lambda j: self.inbox[:RING_BYTES] if r == 0 else self.inbox[:self.payload_bytes(tmap[j])])

    def run_p2p(self, sched, jobs, fresh):
        """The ring over NVLink mailboxes: span r's wire quantizer stores job
        j's codes/scales straight into span r+1's slot, a signal kernel
        publishes it, span r+1's stream waits on it -- no host sync, no NCCL."""
        import torch

        from paper_2209_01188_b200 import _lib
        from paper_2209_01188_b200.pipeline import DevPtr

        r, N, ring = self.rank, self.world, self.ring
        st = _lib.stream_ptr(torch.cuda.current_stream())

        def views(addr, t):
            n = t * self.B * self.d
            return DevPtr(addr), DevPtr(addr + -(-n // 16) * 16)

        for j, t in jobs:
            src, dst = sched.recv_from(j), sched.send_to(j)
            if src is not None:
                ring.wait(j, st)
            n = t * self.B
            seqs = self.seqs[j % self.S]
            if dst is not None and r < N - 1:
                oc, os_ = views(ring.peer_slot(j), t)
            else:
                oc, os_ = self.views(self.outbox, t)
            if r == 0:
                self.span.step_codes(seqs, [t] * self.B, in_f32=self._input(j, n), out_codes=oc, out_scales=os_,
                                     out_f32=self.out[:n])
            else:
                ic, is_ = views(ring.local_slot(j), t)
                self.span.step_codes(seqs, [t] * self.B, in_codes=ic, in_scales=is_, out_codes=oc, out_scales=os_,
                                     out_f32=self.out[:n])
            self.launches += self.span.last_launches + (1 if src is not None else 0) + (1 if dst is not None else 0)
            if fresh:
                for s in seqs:
                    self.span.release(s)
            if dst is not None:
                # forward edge: job j's payload; ring back-edge (last span -> span 0):
                # orders the session's next step j + S (stand-in for the client's head)
                ring.signal(j if r < N - 1 else j + self.S, st)

    def timed(self, lens, clk_index=None):
        """Run one phase between barriers; returns (max-over-ranks ms, launches, clocks)."""
        import torch

        self.barrier()
        self.launches = 0
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = ClockSampler(self.local if clk_index is None else clk_index)
        with clk:
            start.record()
            self.phase(lens)
            stop.record()
            self.barrier()
        ms = start.elapsed_time(stop)
        t = torch.tensor([ms], device=self.dev)
        if self.dist:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item()), self.launches, clk.summary()

    def prefill(self, T0):
        lens, left = [], T0
        per = max(1, self.chunk // self.B)
        while left > 0:
            lens.append(min(per, left))
            left -= lens[-1]
        self.phase(lens)


# ------------------------------------------------------------------ sub-records


def c2_record(args):
    """Config 2: BLOOM-560M shape, all 24 blocks on one GPU, int8,
    128-token prefix then batch-1 decode; steps/s and the fraction of the
    per-step HBM roofline (0.317 GB at T=128 + 0.013 GB KV)."""
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg = SHAPES["bloom-560m"]
    span = BlockSpan(cfg, 0, cfg.n_layers, int8=True, page_tokens=64, n_pages=8, max_tokens=128, max_seqs=2)
    span.generate_weights(args.seed)
    seq = span.new_sequence()
    g = torch.Generator(device="cuda").manual_seed(3)
    prompt = torch.randn(128, cfg.hidden, device="cuda", generator=g) * 0.05
    x1 = torch.randn(1, cfg.hidden, device="cuda", generator=g) * 0.05
    out = torch.empty_like(x1)
    span.step([(seq, prompt)])
    K, W = max(args.steps, 50), max(args.warmup, 5)
    for _ in range(W):
        span.step([(seq, x1)], out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        span.step([(seq, x1)], out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    ctx = 128 + W + K // 2
    w, kv = bytes_per_step(cfg, [ctx])
    peak, _ = measured_peaks()
    ceiling_ms = (w + kv) / (peak * 1e9) * 1e3
    span.close()
    return {"metric": "BLOOM-560M int8 decode steps/s (b=1)", "value": 1e3 / ms, "unit": "steps/s",
            "ms_per_step": ms, "us_per_block": 1e3 * ms / cfg.n_layers, "ctx": ctx,
            "bytes_per_step": w + kv, "roofline_frac": ceiling_ms / ms,
            "note": "24 blocks h=1024 on one GPU, 128-token prefix, batch-1 decode timed with CUDA events"}


def f2_record(args):
    """SURVEY §8 f2 (BACKWARD, server.py:431-450): one 512-position row back
    through two 176B-shape blocks (tape-less recompute + backward, int8
    matrices on tcgen05, attention on 3xTF32 mma). Per block and row: 2 t 20 h^2
    useful matmul flops (recompute qkv/wo/mlp_in 8 h^2 weights, backward all
    four matrices 12 h^2)."""
    import torch

    from paper_2209_01188_b200.model import SHAPES
    from paper_2209_01188_b200.span import BlockSpan

    cfg, L, t = SHAPES["bloom-176b"], 2, 512
    span = BlockSpan(cfg, 0, L, int8=True, page_tokens=64, n_pages=t // 64 + 4, max_tokens=256, max_seqs=8)
    span.generate_weights(args.seed)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(1, t, cfg.hidden, device="cuda", generator=g) * 0.05
    gr = torch.rand(1, t, cfg.hidden, device="cuda", generator=g) * 2 - 1
    _, tape = span.forward(x, tape=True)
    span.backward(tape, gr)  # warm-up: workspace arena, kernel setup
    torch.cuda.synchronize()
    reps = 4
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = span.backward(tape, gr)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps / L
    finite = bool(torch.isfinite(out).all())
    span.close()
    del tape, out
    useful = 2.0 * t * 20 * cfg.hidden ** 2 / (ms / 1e3) / 1e12
    bf16 = measured_tflops()
    return {"metric": "BLOOM-176B BACKWARD positions/s per block (one 512-position row)", "value": t / (ms / 1e3),
            "unit": "positions/s", "ms_per_block": ms, "rows": 1, "t": t, "blocks": L, "finite": finite,
            "useful_matmul_tflops": useful, "tensor_frac_vs_bf16_dense": useful / bf16 if bf16 else None,
            "note": "tape-less recompute + backward per block; int8 matrices on the tcgen05 GEMM (3 int8 digit "
                    "columns per position: issued int8 ops = 3x useful), attention products on 3xTF32 mma.sync"}


def b32_record(pl, args, cfg):
    """BASELINE's tokens/s (b=32): each micro-batch is 32 batch-1 sessions
    stepped together (one launch sequence per block for all 32 tokens)."""
    B, T = 32, args.b32_ctx
    pl.set_batch(B)
    T0 = T - (args.warmup + args.steps) - 1
    lens, left = [], T0
    while left > 0:
        lens.append(min(pl.chunk // B, left))
        left -= lens[-1]
    pl.phase(lens)
    pl.phase([1] * args.warmup)
    ms, launches, clk = pl.timed([1] * args.steps)
    N, S, K = pl.world, pl.S, args.steps
    tokens = K * S * B
    w, kv = bytes_per_step(cfg, [T0 + args.warmup + K // 2] * B)  # one micro-batch through all blocks
    peak, _ = measured_peaks()
    # every GPU streams its span's weights + its KV once per micro-batch step
    agg_ceiling_s = (w / N + kv / N) / (peak * 1e9)
    step_s = (ms / 1e3) / (K * S)
    pl.set_batch(args.batch)
    return {"metric": METRIC_B.format(model=model_label(args.shape), b=B), "value": tokens / (ms / 1e3),
            "unit": "tokens/s", "sessions": S * B, "ctx_end": T, "ms_per_microbatch_step": step_s * 1e3 * N,
            "bytes_per_step": w + kv, "roofline_frac": agg_ceiling_s / step_s, "gpu_launches": launches,
            "clocks": clk, "note": f"{S} micro-batch(es) x {B} sessions, context {T0}->{T}; roofline = every GPU "
                                   f"streaming its span's int8 weights + KV once per micro-batch step"}


def forward_record(pl, args, cfg):
    """C5-style FORWARD: rows of 512 tokens (server.py:411-429 semantics,
    cache-less, no tape) through the pipeline, S rows in flight."""
    import torch

    rows = max(1, args.forward_rows) * pl.S
    pl.set_batch(1)
    per_mb = rows // pl.S
    pl.span.profile(True)
    pl.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pl.phase([512] * per_mb, fresh=True)
    e1.record()
    pl.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device=pl.dev)
    if pl.dist:
        pl.dist.all_reduce(t, op=pl.dist.ReduceOp.MAX)
    ms = float(t.item())
    g_ms, g_n, g_ops = pl.span.profile_read(5)
    a_ms, _, _ = pl.span.profile_read(pl.span.PROF_ATTN)
    pl.span.profile(False)
    tokens = rows * 512
    useful = 2.0 * tokens * cfg.n_layers * 12 * cfg.hidden * cfg.hidden
    return {"rows": rows, "tokens_per_row": 512, "ms": ms, "tokens_per_s": tokens / (ms / 1e3),
            "useful_tflops_per_gpu": useful / pl.world / (ms / 1e3) / 1e12,
            "tcgen05_gemm": {"launches": g_n, "ms": g_ms,
                             "useful_tflops": g_ops / 3.0 / max(g_ms, 1e-9) / 1e9 if g_n else None},
            "tcgen05_share": g_ms / ms, "attention_share": a_ms / ms,
            "peak_tflops_dense_bf16_measured": measured_tflops(),
            "note": "C5 rows of 512 tokens through all 70 blocks, one 512-token job per row, rows pipelined over "
                    "the spans; useful flops = 2*tokens*12h^2 per block (matmuls only); the event-profiled "
                    "pass that gives the tcgen05/attention shares is the timed one"}


def _e2e_out_of_process(address, S, prefill_msgs, step_msgs, per_frame, T0, W, K, ctx):
    """Run the e2e client sessions in a separate process (`bench.py
    --e2e-client`); returns (wall seconds, errors, description) or (None, ...)
    when that process cannot be used."""
    import pickle
    import tempfile

    proc, spec = None, None
    try:
        with tempfile.NamedTemporaryFile("wb", suffix=".pkl", delete=False) as f:
            pickle.dump({"address": address, "S": S, "prefill": prefill_msgs, "steps_msgs": step_msgs,
                         "per_frame": per_frame, "T0": T0, "W": W, "K": K, "ctx": ctx}, f)
            spec = f.name
        proc = subprocess.Popen([sys.executable, os.path.abspath(__file__), "--e2e-client", spec],
                                stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
        line = proc.stdout.readline()
        if line.strip() != "READY":
            raise RuntimeError(f"client process: {line!r}")
        proc.stdin.write("GO\n")
        proc.stdin.flush()
        res = json.loads(proc.stdout.readline())
        proc.wait(timeout=60)
        return res["wall"], res["errors"], "a separate client process, one thread per session"
    except Exception as e:  # noqa: BLE001
        print(f"[e2e] client process unavailable ({e!r}); clients on threads of this process", file=sys.stderr)
        if proc is not None and proc.poll() is None:
            proc.kill()
        return None, [], None
    finally:
        if spec:
            try:
                os.unlink(spec)
            except OSError:
                pass


def e2e_record(pl, args, cfg, T0):
    """The headline metric through the server's public API: S client sessions
    (threads of a separate client process, as the reference's clients are
    separate programs; threads of this process if that process fails) each
    open a session, prefill T0 tokens with int8 STEP frames, then send
    W + K one-token STEP frames (int8 TensorMsg built on the host) and read the
    replies. N=1: ServerNode on the resident span; N>1: the box front end (one
    ServerEntry [0, 70), rank 0 accepts TCP, the hops stay on the GPUs)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2209_01188_b200.box import BoxFrontEnd, BoxPlan, RankState, payload_bytes, serve_rank, FMT_F32
    from paper_2209_01188_b200.server import ServerConfig, ServerNode
    from paper_2209_01188_b200 import codec

    N, K, W = pl.world, args.steps, args.warmup
    S = pl.S * args.batch  # client sessions: the headline's micro-batches x batch-1 sessions each
    unit = UNIT if args.batch == 1 else "tokens/s"
    pl.set_batch(1)
    for grp in pl.seqs:
        for s in grp:
            pl.span.release(s)
    scfg = ServerConfig(seed=args.seed, model=cfg, blocks=(0, cfg.n_layers), quantize="both", capacity=max(S, 4),
                        cache_budget_tokens=cfg.n_layers * (args.ctx + 64) * (S + 1), max_batch_tokens=pl.chunk,
                        measure_steps=3, page_tokens=64, device=pl.local)
    node = None
    if N == 1:
        node = ServerNode(scfg, span=pl.span).start()
    else:
        gloo = dist.new_group(backend="gloo")
        plan = BoxPlan(scfg, N)
        from paper_2209_01188_b200.pipeline import P2PRing

        ring = P2PRing(pl.rank, N, plan.in_flight, payload_bytes(pl.chunk, cfg.hidden, FMT_F32), pl.local, dist)
        state = RankState(plan, pl.rank, pl.span, ring, dist, group=gloo, owns_span=False)
        if pl.rank > 0:
            serve_rank(plan, pl.rank, dist, state=state)
            return None
        node = BoxFrontEnd(scfg, N, dist, state=state).start()
    rng = np.random.default_rng(11)
    d = cfg.hidden
    # a TensorMsg is capped at 64 MiB counted as f32 (transport/wire.py:93-94, even for int8), i.e. 1170
    # tokens at h=14336: the client sends a long prompt as consecutive STEPs
    per_frame = max(1, (64 * 1024 * 1024) // (4 * d) - 1)
    prefill_msgs = [codec.encode_tensor(rng.standard_normal((min(per_frame, T0 - p), d)).astype(np.float32) * 0.05,
                                        codec.ENC_INT8) for p in range(0, T0, per_frame)]
    step_msgs = [codec.encode_tensor(rng.standard_normal((1, d)).astype(np.float32) * 0.05, codec.ENC_INT8)
                 for _ in range(8)]
    wall, errors, clients = _e2e_out_of_process(node.address, S, prefill_msgs, step_msgs, per_frame, T0, W, K,
                                                args.ctx)
    if wall is None:  # the client process failed to start or report: the same sessions on threads here
        clients = "threads of the bench process"
        ready, go = threading.Barrier(S + 1), threading.Event()
        ts, times, errors = _client_sessions(node.address, S, prefill_msgs, step_msgs, per_frame, T0, W, K,
                                             args.ctx, ready, go)
        try:
            ready.wait(timeout=900)
        except threading.BrokenBarrierError:
            pass
        t_start = time.perf_counter()
        go.set()
        for t in ts:
            t.join()
        wall = time.perf_counter() - t_start
    if os.environ.get("PB_SERVER_TIMING") == "1" and node.timing:  # diagnostic: per-STEP host split (ms)
        cols = list(zip(*node.timing[-K * S:]))
        print("[e2e] STEP decode / compute / encode ms (median):",
              [round(1e3 * statistics.median(c), 3) for c in cols], file=sys.stderr, flush=True)
        stt = getattr(node, "step_timing", None)
        if stt:
            print("[e2e] box STEP decode / ring / encode ms (median):",
                  [round(1e3 * statistics.median(c), 3) for c in zip(*stt[-K * S:])], file=sys.stderr, flush=True)
        bt = getattr(node.sched, "timing", None)
        if bt:
            d = [[b - a for a, b in zip(t, t[1:])] for t in bt[-K * S:]]
            print("[e2e] box job send / rank-0 launch / egress launch / ring+egress ms (median):",
                  [round(1e3 * statistics.median(c), 3) for c in zip(*d)], file=sys.stderr, flush=True)
    node.stop()
    if errors:
        return {"error": errors[0]}
    step_bytes = len(step_msgs[0])
    return {"value": K * S / wall, "unit": unit, "h2d_bytes_per_step": step_bytes, "d2h_bytes_per_step": step_bytes,
            "wall_s": wall, "sessions": S, "ctx_end": T0 + W + K,
            "path": ("TCP STEP frames (int8 TensorMsg) -> " + ("ServerNode" if N == 1 else
                     f"box front end over {N} GPUs (one ServerEntry [0, 70), peer-memory hops)") +
                     f" -> reply frames read by the clients ({clients}); prefill via int8 STEPs of <= 1169 tokens "
                     "per session, untimed")}


# ------------------------------------------------------------------ main


def run_ours(args):
    import torch

    from paper_2209_01188_b200.model import SHAPES

    cfg = SHAPES[args.shape]
    label = model_label(args.shape)
    metric, unit = ((METRIC.format(model=label), UNIT) if args.batch == 1
                    else (METRIC_B.format(model=label, b=args.batch), "tokens/s"))
    rank0 = int(os.environ.get("RANK", "0")) == 0
    c2 = None
    if not args.no_c2 and rank0 and args.shape == "bloom-176b":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        c2 = c2_record(args)  # before the 176B span: HBM is nearly full with it
        torch.cuda.empty_cache()
    f2 = None
    if not args.no_f2 and rank0 and args.shape == "bloom-176b":
        f2 = f2_record(args)
        torch.cuda.empty_cache()
    pl = Pipeline(args, cfg)
    S, N, rank, B = pl.S, pl.world, pl.rank, pl.B
    K, W = args.steps, args.warmup
    T0 = args.ctx - (W + 2 * K) - 1
    if T0 < 1:
        raise SystemExit("--ctx too small for warmup+steps")
    # ---- prefill every session to T0 through the pipeline (untimed; tcgen05 GEMM device time recorded)
    t_pf = time.perf_counter()
    pl.span.profile(True)
    if args.synthetic_kv:
        for grp in pl.seqs:
            for s in grp:
                pl.span.reserve(s, T0)
                s.length = T0
    else:
        pl.prefill(T0)
    torch.cuda.synchronize()
    pf_s = time.perf_counter() - t_pf
    tc_ms, tc_n, tc_flop = pl.span.profile_read(5)
    pl.span.profile(False)
    # ---- warmup + timed decode (device-resident inputs)
    pl.phase([1] * W)
    ms_max, launches, clocks = pl.timed([1] * K)
    # ---- live per-kernel device times (CUDA events around every launch on the
    # launching stream) over a second, identical pass of K steps, outside the
    # value's timed region so the events do not perturb it
    pl.span.profile(True)
    pl.phase([1] * K)
    pl.barrier()
    gemv = pl.span.profile_read(pl.span.PROF_GEMV)
    attn = pl.span.profile_read(pl.span.PROF_ATTN)
    pro = pl.span.profile_read(pl.span.PROF_PROLOGUE)
    codec_p = pl.span.profile_read(pl.span.PROF_CODEC)
    pl.span.profile(False)
    value = K * S * B / (ms_max / 1e3)  # session-steps (= tokens) per second over all GPUs
    # ---- sub-records
    e2e = None if args.no_e2e else e2e_record(pl, args, cfg, T0)
    b32 = None if args.no_b32 else b32_record(pl, args, cfg)
    fwd = forward_record(pl, args, cfg) if args.forward_rows > 0 else None
    if rank != 0:
        if pl.dist:
            pl.dist.barrier()
            pl.dist.destroy_process_group()
        return
    peak, peak_kind = measured_peaks()
    g_ms, g_n, g_b = gemv
    achieved = (g_b / g_n) / ((g_ms / g_n) / 1e3) / 1e9 if g_n else 0.0
    traffic = committed_traffic()
    w_bytes, kv_bytes = bytes_per_step(cfg, [args.ctx - K // 2] * (S * B))
    step_s = (ms_max / 1e3) / (K * S)
    seq_ceiling = (w_bytes + kv_bytes / S) / (peak * 1e9)
    agg_ceiling = (w_bytes / N + kv_bytes / N / S) / (peak * 1e9)
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": N, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "int8 weights x int8-digit activations (22-bit fixed point, exact s32 accumulate); fp16 KV; f32 residual",
        "data": "synthetic (gen_checkpoint seed 42 weights generated on device; random embedding-like inputs)",
        "config": {"workload": f"{args.shape} ({cfg.n_layers} blocks, h={cfg.hidden}) int8 decode, {S} micro-batch(es) "
                               f"of {B} batch-1 session(s) pipelined over {N} GPU span(s) {pl.ranges}, "
                               f"context {T0}->{args.ctx}",
                   "sessions": S * B, "batch_per_microbatch": B, "ctx_end": args.ctx, "prefill_tokens": T0,
                   "l2": "weights stream 172.7 GB per step >> 126 MB L2 (no flush needed)",
                   "parallelism": f"pipeline{N} (block spans)",
                   "hop": "none" if N == 1 else ("p2p" if pl.ring is not None else "nccl")},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": traffic.get("gemv_i8_bytes_per_launch") if traffic else None,
                     "kernel": "k_gemv_i8 (int8 GEMV, all 4 matrices of every block)",
                     "launches": g_n, "avg_launch_us": 1e3 * g_ms / max(g_n, 1),
                     "algorithmic_bytes_per_launch": g_b / max(g_n, 1), "peak_source": peak_kind},
        "step_roofline": {"bytes_per_step": w_bytes + kv_bytes / S, "sequential_frac": seq_ceiling / (ms_max / 1e3 / K),
                          "aggregate_frac": agg_ceiling / step_s,
                          "kernel_share": {"gemv": g_ms / ms_max, "attention": attn[0] / ms_max,
                                           "prologue": pro[0] / ms_max, "codec": codec_p[0] / ms_max}},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "b32": b32,
        "c2": c2,
        "f2": f2,
        "setup_s": {"weights_gen_quant": pl.gen_s, "prefill": pf_s},
        "prefill": {"tokens": T0 * S * B, "wall_s": pf_s, "tokens_per_s_wall": T0 * S * B / max(pf_s, 1e-9),
                    "tcgen05_gemm": {"launches": tc_n, "ms": tc_ms,
                                     "achieved_int8_tops": tc_flop / max(tc_ms, 1e-9) / 1e9 if tc_n else None,
                                     "useful_tflops": tc_flop / 3.0 / max(tc_ms, 1e-9) / 1e9 if tc_n else None,
                                     "peak_int8_tops_dense_nominal": 4500.0,
                                     "peak_tflops_dense_bf16_measured": measured_tflops(),
                                     "note": "kind::i8 ops issued (3 int8 digit columns per token); useful = "
                                             "2*M*K*tokens of the reference matmul"}},
        "forward": fwd,
        "device_bytes": pl.span.device_bytes,
    }
    if not args.no_cpu_baseline and N == 1:
        sample, ncores = cpu_block_sample(cfg, args.ctx)
        sample.step_seconds()
        all_t = cpu_step_seconds(sample, 2)
        one_t = cpu_step_seconds(sample, 1, threads=1)
        line["cpu_baseline"] = {
            "value": 1.0 / (all_t * cfg.n_layers), "unit": unit, "cores": ncores, "kind": "port",
            "sample": f"oracle port of block_forward(qw) (f32 KV concat, dequantized-matrix matmuls) for 1 "
                      f"{args.shape} block, decode t=1 at context {args.ctx}, best of 2, extrapolated x{cfg.n_layers}",
            "one_thread": {"value": 1.0 / (one_t * cfg.n_layers), "block_s": one_t},
            "all_threads_block_s": all_t, **cpu_info()}
    print(json.dumps(line), flush=True)
    if pl.dist:
        pl.dist.barrier()
        pl.dist.destroy_process_group()


def _client_sessions(address, S, prefill_msgs, step_msgs, per_frame, T0, W, K, ctx, ready, go):
    """S client sessions on threads: open, prefill T0 tokens (int8 STEP frames of
    <= per_frame rows), W warm-up steps, then (after ready/go) K timed one-token
    STEP frames each. Returns (per-session seconds, errors)."""
    from paper_2209_01188_b200 import codec
    from paper_2209_01188_b200.client import SpanClient

    times, errors = [0.0] * S, []

    def client(i):
        c = SpanClient(address, codec.ENC_INT8, timeout_ms=600_000)
        try:
            sid = c.open_session(ctx)
            pos = 0
            for msg in prefill_msgs:
                c.step_raw(sid, pos, msg)
                pos += min(per_frame, T0 - pos)
            for k in range(W):
                c.step_raw(sid, pos, step_msgs[k % len(step_msgs)])
                pos += 1
            ready.wait()
            go.wait()
            t0 = time.perf_counter()
            for k in range(K):
                reply = c.step_raw(sid, pos, step_msgs[k % len(step_msgs)])
                codec.parse_tensor(reply)  # the host reads the int8 reply (codes + scales)
                pos += 1
            times[i] = time.perf_counter() - t0
            c.close_session(sid)
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))
            try:
                ready.abort()
            except Exception:  # noqa: BLE001
                pass
        finally:
            c.close()

    ts = [threading.Thread(target=client, args=(i,)) for i in range(S)]
    for t in ts:
        t.start()
    return ts, times, errors


def e2e_client_process():
    """`bench.py --e2e-client SPEC`: the e2e clients in their own process (as the
    reference's clients are), so the server's threads do not share an
    interpreter lock with them. Prints READY after every session's prefill and
    warm-up, starts the timed steps on a line from stdin, prints the result."""
    import pickle

    with open(sys.argv[2], "rb") as f:
        spec = pickle.load(f)
    ready, go = threading.Barrier(spec["S"] + 1), threading.Event()
    ts, times, errors = _client_sessions(spec["address"], spec["S"], spec["prefill"], spec["steps_msgs"],
                                         spec["per_frame"], spec["T0"], spec["W"], spec["K"], spec["ctx"], ready, go)
    try:
        ready.wait(timeout=900)
    except threading.BrokenBarrierError:
        pass
    print("READY", flush=True)
    sys.stdin.readline()
    t_start = time.perf_counter()
    go.set()
    for t in ts:
        t.join()
    wall = time.perf_counter() - t_start
    print(json.dumps({"wall": wall, "errors": errors}), flush=True)


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--e2e-client":
        e2e_client_process()
        return
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
