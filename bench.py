"""Headline benchmark: BLOOM-176B-shape int8 decode steps/s (BASELINE.json).

Workload (N GPUs, one process per GPU): the 70-block 176B-shape model
(h=14336, H=112, int8 weights generated on device from the reference's
SplitMix64 streams) is split into N contiguous block spans, one per GPU
(N=1: all 70 blocks on one B200). N batch-1 sessions are in flight (one per
pipeline stage, "weak" scaling: per-GPU work is constant), each decoding at a
context that ends at --ctx (default 2048). A step is one decode token of one
session through all 70 blocks; span-to-span hops carry the hidden state as
the reference's blockwise int8 wire codec over NCCL send/recv (the last span
hands the result back to span 0, which closes the ring for the next token).

value = session-steps/s over all GPUs (b=1 per session) measured with CUDA
events between barriers, max over ranks. e2e = same metric through the
server's STEP handler with host bytes in/out (N=1) or with pinned-host
ingress/egress copies at the pipeline ends (N>1).

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


def model_label(shape: str) -> str:
    return shape.upper()  # bloom-176b -> BLOOM-176B
RING_BYTES = 64
UNIT = "steps/s"


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
    p.add_argument("--prefill-chunk", type=int, default=240)
    p.add_argument("--batch", type=int, default=1, help="batch-1 sessions per pipeline micro-batch")
    p.add_argument("--hop", default="p2p", choices=["p2p", "nccl"],
                   help="span-to-span hop: NVLink peer-memory mailboxes (pb_hop.cu) or NCCL send/recv")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--synthetic-kv", action="store_true", help="skip the real prefill (KV content is synthetic)")
    p.add_argument("--forward-rows", type=int, default=2, help="rows of the FORWARD sample (C5 shape: 512 tokens each)")
    return p.parse_args()


# ------------------------------------------------------------------ helpers


from paper_2209_01188_b200.pipeline import split_blocks  # noqa: E402


def bytes_per_step(cfg, ctx_tokens_per_session):
    """sum_blocks [12h^2 codes + 7h*4 scales + 13h*4 bias/LN]
    + sum_sessions sum_blocks 2*T*h*2 (fp16 K+V)."""
    h, L = cfg.hidden, cfg.n_layers
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
            self._stop.wait(0.2)

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
        return float(d["hbm_gbs"]), "measured"
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


def cpu_block_sample(cfg, ctx_sample):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import cpu_baseline

    return cpu_baseline.BlockSample(cfg.hidden, cfg.n_heads, ctx_sample, cfg.mlp_ratio), cpu_baseline.cores()


def run_reference(args):
    """--impl reference: the reference's CPU arithmetic (oracle port of
    block_forward(qw) / matmul_mixed) on the host cores; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2209_01188_b200.model import SHAPES

    cfg = SHAPES[args.shape]
    ctx_sample = 128
    sample, ncores = cpu_block_sample(cfg, ctx_sample)
    for _ in range(args.warmup):
        sample.step_seconds()
    ts = [sample.step_seconds() for _ in range(args.steps)]
    per_block = min(ts)  # best case for the CPU (OpenBLAS timings are noisy)
    value = 1.0 / (per_block * cfg.n_layers)
    desc = (f"1 block of the {args.shape} shape, int8 decode t=1 at context {ctx_sample} (oracle port of "
            f"quant.py matmul_mixed + model.py block_forward, random codes), x{cfg.n_layers} blocks extrapolated")
    line = {
        "impl": "reference", "metric": METRIC.format(model=model_label(args.shape)), "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_block * cfg.n_layers * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": f"{args.shape} int8 decode b=1 (CPU reference arithmetic)",
                                        "ctx": ctx_sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU pipeline


class Pipeline:
    """One span of the 70-block model per GPU; jobs follow the deadlock-free
    ring schedule of paper_2209_01188_b200.pipeline (grouped NCCL send/recv of
    the int8 wire payload: codes then f32 scales in one byte buffer)."""

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

            dist.init_process_group("nccl", device_id=self.dev, timeout=datetime.timedelta(seconds=180))
        self.dist = dist if self.world > 1 else None
        self.S = self.world  # micro-batches in flight (one per pipeline stage)
        self.B = args.batch  # batch-1 sessions per micro-batch
        self.chunk = max(1, args.prefill_chunk // self.B)  # prefill positions per sequence per step
        self.ranges = split_blocks(cfg.n_layers, self.world)
        s, e = self.ranges[self.rank]
        pages_per_seq = -(-min(cfg.max_seq, args.ctx + 64) // 64)  # KV pool sized for the benchmarked context
        t0 = time.perf_counter()
        self.span = BlockSpan(cfg, s, e, int8=True, page_tokens=64, n_pages=self.S * self.B * pages_per_seq + 2,
                              max_tokens=max(self.chunk * self.B, 512), max_seqs=max(self.B, 2), device=self.local)
        self.span.generate_weights(args.seed)
        torch.cuda.synchronize()
        self.gen_s = time.perf_counter() - t0
        self.seqs = [[self.span.new_sequence() for _ in range(self.B)] for _ in range(self.S)]
        d = cfg.hidden
        self.d = d
        cap = self.payload_bytes(self.chunk)
        self.inbox = torch.empty(cap, dtype=torch.uint8, device=self.dev)
        self.outbox = torch.empty(cap, dtype=torch.uint8, device=self.dev)
        self.out = torch.empty(self.chunk * self.B, d, dtype=torch.float32, device=self.dev)
        g = torch.Generator(device=self.dev)
        g.manual_seed(7)
        self.inputs = torch.randn(64, d, generator=g, device=self.dev) * 0.05  # embedding-like rows
        self.launches = 0
        self.total_jobs = 0
        self.jobtimes = [] if os.environ.get("PB_BENCH_JOBTIMES") else None  # diagnostic: per-job device times
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

    def payload_bytes(self, t):
        n = t * self.B * self.d
        return -(-n // 16) * 16 + 4 * (-(-n // 64))

    def views(self, buf, t):
        n = t * self.B * self.d
        off = -(-n // 16) * 16
        return buf[:n].view(__import__("torch").int8), buf[off:off + 4 * (-(-n // 64))].view(__import__("torch").float32)

    def barrier(self):
        import torch

        torch.cuda.synchronize()
        if self.dist:
            self.dist.barrier()
        torch.cuda.synchronize()

    def run(self, jobs, x_for=None, host_in=None, host_out=None, sync_out=False):
        """jobs: [(job id, new positions t per sequence)]; x_for(j, n) -> span-0 input rows."""
        import torch

        from paper_2209_01188_b200.pipeline import RingSchedule, run_jobs, torch_exchange

        sched = RingSchedule(self.rank, self.world, self.S, self.total_jobs)
        tmap = dict(jobs)
        r, N = self.rank, self.world

        jt = self.jobtimes

        def step(j, inbox):
            if jt is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                jt.append(e)
            t = tmap[j]
            n = t * self.B
            seqs = self.seqs[j % self.S]
            outbox = self.outbox
            oc, os_ = self.views(outbox, t)
            if inbox is None or r == 0:  # span 0: fresh input (a received ring payload only orders the step)
                if host_in is not None:
                    self.out[:n].copy_(host_in[:n], non_blocking=True)
                    inp = self.out[:n]
                elif x_for is not None:
                    inp = x_for(j, n)
                else:
                    inp = self.inputs[j % 64: j % 64 + 1].expand(n, self.d).contiguous()
                self.span.step_codes(seqs, [t] * self.B, in_f32=inp, out_codes=oc, out_scales=os_, out_f32=self.out[:n])
            else:
                ic, is_ = self.views(inbox, t)
                self.span.step_codes(seqs, [t] * self.B, in_codes=ic, in_scales=is_, out_codes=oc, out_scales=os_,
                                     out_f32=self.out[:n])
            self.launches += self.span.last_launches
            if jt is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                jt.append(e)
            if r == N - 1 and host_out is not None:
                host_out[:n * self.d].copy_(oc, non_blocking=True)
                if sync_out:
                    torch.cuda.current_stream().synchronize()  # result readable on the host
            if r == N - 1:
                # ring back-edge: only orders span 0's next step of this session
                # (stand-in for the client's LM head); fixed size, so prefill
                # chunks and decode steps of different t always match
                return outbox[:RING_BYTES]
            return outbox[:self.payload_bytes(t)]

        if self.ring is not None:
            self.run_p2p(sched, jobs, tmap, x_for, host_in, host_out, sync_out)
            return
        run_jobs(sched, [j for j, _ in jobs], step, torch_exchange,
                 lambda j: self.inbox[:RING_BYTES] if r == 0 else self.inbox[:self.payload_bytes(tmap[j])])

    def run_p2p(self, sched, jobs, tmap, x_for, host_in, host_out, sync_out):
        """The same ring over NVLink mailboxes: span r's wire quantizer stores
        job j's codes/scales straight into span r+1's slot, a signal kernel
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
                if host_in is not None:
                    self.out[:n].copy_(host_in[:n], non_blocking=True)
                    inp = self.out[:n]
                elif x_for is not None:
                    inp = x_for(j, n)
                else:
                    inp = self.inputs[j % 64: j % 64 + 1].expand(n, self.d).contiguous()
                self.span.step_codes(seqs, [t] * self.B, in_f32=inp, out_codes=oc, out_scales=os_, out_f32=self.out[:n])
            else:
                ic, is_ = views(ring.local_slot(j), t)
                self.span.step_codes(seqs, [t] * self.B, in_codes=ic, in_scales=is_, out_codes=oc, out_scales=os_,
                                     out_f32=self.out[:n])
            self.launches += self.span.last_launches + (1 if src is not None else 0) + (1 if dst is not None else 0)
            if r == N - 1 and host_out is not None:
                host_out[:n * self.d].copy_(oc, non_blocking=True)
                if sync_out:
                    torch.cuda.current_stream().synchronize()
            if dst is not None:
                # forward edge: job j's payload; ring back-edge (last span -> span 0):
                # orders the session's next step j + S (stand-in for the client's head)
                ring.signal(j if r < N - 1 else j + self.S, st)


def run_ours(args):
    import torch

    from paper_2209_01188_b200.model import SHAPES

    cfg = SHAPES[args.shape]
    label = model_label(args.shape)
    metric, unit = ((METRIC.format(model=label), UNIT) if args.batch == 1
                    else (METRIC_B.format(model=label, b=args.batch), "tokens/s"))
    pl = Pipeline(args, cfg)
    S, N, rank, B = pl.S, pl.world, pl.rank, pl.B
    K, W = args.steps, args.warmup
    T0 = args.ctx - (W + 2 * K) - (0 if args.no_e2e else K) - 1
    if T0 < 1:
        raise SystemExit("--ctx too small for warmup+steps")
    # ---- prefill every session to T0 through the pipeline (untimed)
    t_pf = time.perf_counter()
    pl.span.profile(True)  # prefill runs the tcgen05 GEMM: record its live device time
    if args.synthetic_kv:
        for grp in pl.seqs:
            for s in grp:
                pl.span._reserve(s, T0)
                s.length = T0
    else:
        chunks = []
        left = T0
        while left > 0:
            c = min(pl.chunk, left)
            chunks.append(c)
            left -= c
        # job order: for each chunk round, every session (keeps the ring pattern)
        jobs = [(ci * S + m, c) for ci, c in enumerate(chunks) for m in range(S)]
        pl.total_jobs = len(jobs) + S * (W + 2 * K + (0 if args.no_e2e else K))
        # all prefill jobs, then decode jobs continue numbering
        pl.run(jobs, x_for=lambda j, n: pl.inputs[:n] if n <= 64 else torch.randn(n, cfg.hidden, device=pl.dev) * 0.05)
        jbase = len(jobs)
    torch.cuda.synchronize()
    pf_s = time.perf_counter() - t_pf
    tc_ms, tc_n, tc_flop = pl.span.profile_read(5)
    pl.span.profile(False)
    if args.synthetic_kv:
        jbase = 0
        pl.total_jobs = S * (W + 2 * K + (0 if args.no_e2e else K))
    # ---- warmup decode
    pl.run([(jbase + i, 1) for i in range(W * S)])
    jbase += W * S
    # ---- timed decode (device-resident inputs)
    pl.barrier()
    pl.launches = 0
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(pl.local) as clk:
        start.record()
        pl.run([(jbase + i, 1) for i in range(K * S)])
        stop.record()
        pl.barrier()
    jbase += K * S
    ms = start.elapsed_time(stop)
    if pl.jobtimes is not None:
        ev = pl.jobtimes[-2 * K * S:]
        busy = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(K * S)]
        gaps = [ev[2 * i - 1].elapsed_time(ev[2 * i]) for i in range(1, K * S)]
        print(f"[rank {rank}] job busy ms mean {statistics.mean(busy):.3f} max {max(busy):.3f} | "
              f"gap ms mean {statistics.mean(gaps):.3f} max {max(gaps):.3f}", file=sys.stderr, flush=True)
        pl.jobtimes = None
    launches = pl.launches
    # ---- live per-kernel device times (CUDA events around every launch on the
    # launching stream) over a second, identical pass of K steps; kept out of
    # the value's timed region so the events do not perturb it
    pl.span.profile(True)
    pl.run([(jbase + i, 1) for i in range(K * S)])
    pl.barrier()
    jbase += K * S
    gemv = pl.span.profile_read(pl.span.PROF_GEMV)
    attn = pl.span.profile_read(pl.span.PROF_ATTN)
    pro = pl.span.profile_read(pl.span.PROF_PROLOGUE)
    codec_p = pl.span.profile_read(pl.span.PROF_CODEC)
    pl.span.profile(False)
    t = torch.tensor([ms], device=pl.dev)
    if pl.dist:
        pl.dist.all_reduce(t, op=pl.dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = K * S * B / (ms_max / 1e3)  # session-steps (= tokens) per second over all GPUs
    # ---- e2e: host bytes in/out
    e2e = None
    if not args.no_e2e:
        d = cfg.hidden
        host_in = torch.randn(B, d).mul_(0.05).pin_memory()
        host_out = torch.empty(B * d, dtype=torch.int8).pin_memory()
        pl.barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pl.run([(jbase + i, 1) for i in range(K * S)], host_in=host_in if rank == 0 else None,
               host_out=host_out if rank == N - 1 else None, sync_out=True)
        e1.record()
        pl.barrier()
        wall = time.perf_counter() - t0
        te = torch.tensor([max(e0.elapsed_time(e1), wall * 1e3)], device=pl.dev)
        if pl.dist:
            pl.dist.all_reduce(te, op=pl.dist.ReduceOp.MAX)
        e2e = {"value": K * S * B / (float(te.item()) / 1e3), "unit": unit, "h2d_bytes_per_step": 4 * d * B,
               "d2h_bytes_per_step": d * B, "path": "pb_span_step_int8 C-ABI with pinned host ingress (span 0) and "
               "egress of the int8 hidden (last span), " + ("NVLink peer-memory" if pl.ring is not None else "NCCL") + " int8 hops between spans"}
    # ---- FORWARD sample (C5 shape: rows of 512 tokens through this rank's span, tcgen05 path;
    # server.py:411-429 semantics, no tape), timed with CUDA events; each rank its own span
    fwd = None
    if args.forward_rows > 0:
        for grp in pl.seqs:  # decode sessions are done: their KV pages host the FORWARD rows
            for sq in grp:
                pl.span.release(sq)
        rows, t = args.forward_rows, 512
        xb = torch.randn(rows, t, cfg.hidden, device=pl.dev) * 0.05
        pl.span.forward(xb)  # warm-up
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        pl.span.forward(xb)
        f1.record()
        torch.cuda.synchronize()
        f_ms = f0.elapsed_time(f1)
        pl.span.profile(True)  # separate pass: per-kernel shares
        pl.span.forward(xb)
        torch.cuda.synchronize()
        g_ms, g_n, g_ops = pl.span.profile_read(5)
        a_ms, _, _ = pl.span.profile_read(pl.span.PROF_ATTN)
        pl.span.profile(False)
        s0, s1 = pl.ranges[rank]
        useful = 2.0 * rows * t * (s1 - s0) * 12 * cfg.hidden * cfg.hidden
        fwd = {"rows": rows, "tokens_per_row": t, "blocks": s1 - s0, "ms": f_ms,
               "tokens_per_s": rows * t / (f_ms / 1e3), "useful_tflops": useful / (f_ms / 1e3) / 1e12,
               "tcgen05_share": g_ms / f_ms, "attention_share": a_ms / f_ms,
               "note": "FORWARD of rows x 512 tokens through this GPU's span (C5 row shape); useful flops = "
                       "2*tokens*12h^2 per block (matmuls only; profile pass for the shares)"}
    # ---- report (rank 0)
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
    step_s = (ms_max / 1e3) / (K * S)  # one micro-batch step through all blocks
    seq_ceiling = (w_bytes + kv_bytes / S) / (peak * 1e9)  # one micro-batch through all blocks, one GPU busy
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
                   "parallelism": f"pipeline{N} (block spans)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": traffic.get("gemv_i8_bytes_per_launch") if traffic else None,
                     "kernel": "k_gemv_i8 (int8 GEMV, all 4 matrices of every block)",
                     "launches": g_n, "avg_launch_us": 1e3 * g_ms / max(g_n, 1),
                     "algorithmic_bytes_per_launch": g_b / max(g_n, 1), "peak_source": peak_kind},
        # sequential: one session's step latency (each session stepped K times in the timed
        # region) vs all of its bytes through one GPU; aggregate: job throughput vs every GPU
        # streaming its own span's bytes for every micro-batch step
        "step_roofline": {"bytes_per_step": w_bytes + kv_bytes / S, "sequential_frac": seq_ceiling / (ms_max / 1e3 / K),
                          "aggregate_frac": agg_ceiling / step_s,
                          "kernel_share": {"gemv": g_ms / ms_max, "attention": attn[0] / ms_max,
                                           "prologue": pro[0] / ms_max, "codec": codec_p[0] / ms_max}},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
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
        sample, ncores = cpu_block_sample(cfg, 128)
        sample.step_seconds()
        ts = [sample.step_seconds() for _ in range(2)]
        per_block = min(ts)
        line["cpu_baseline"] = {
            "value": 1.0 / (per_block * cfg.n_layers), "unit": unit, "cores": ncores, "kind": "port",
            "sample": f"oracle port of block_forward(qw) for 1 {args.shape} block, decode t=1 at context 128, "
                      f"best of 2, extrapolated x{cfg.n_layers} blocks"}
    print(json.dumps(line), flush=True)
    if pl.dist:
        pl.dist.barrier()
        pl.dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
