"""Two-rank parity check of the NVLink peer-memory hop (pipeline.P2PRing,
pb_hop.cu): 4 blocks split [0,2) on rank 0 and [2,4) on rank 1, S=2 sessions,
a prefill chunk then decode steps around the ring. Rank 1 records every job's
output; rank 0 then replays the same jobs through fresh spans of both halves
in one process (wire codes handed over in HBM) and requires bit-identical
hidden states. With one visible GPU both ranks share it (the mailbox is then a
CUDA IPC mapping within one device -- same code path, no NVLink). The control
plane (handle exchange, barriers) uses gloo; the data path never touches it.
Run under torchrun with 2 processes:

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_check.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    from paper_2209_01188_b200 import _lib
    from paper_2209_01188_b200.model import ModelConfig
    from paper_2209_01188_b200.pipeline import DevPtr, P2PRing, RingSchedule
    from paper_2209_01188_b200.span import BlockSpan

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 2
    gpu = rank % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    dist.init_process_group("gloo")
    cfg = ModelConfig(4, 512, 8, 1024, 256)  # 4 blocks, h=512, 8 heads
    S, d = 2, cfg.hidden
    lens = [16, 1, 1, 1, 1]  # prefill chunk, then decode steps (per session)
    jobs = [(i * S + m, t) for i, t in enumerate(lens) for m in range(S)]
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    inputs = [torch.randn(t, d, generator=g, device=dev) * 0.5 for _, t in jobs]

    def make(lo, hi):
        sp = BlockSpan(cfg, lo, hi, int8=True, page_tokens=16, max_tokens=32, max_seqs=1, device=gpu)
        sp.generate_weights(42)
        return sp

    span = make(2 * rank, 2 * rank + 2)
    seqs = [span.new_sequence() for _ in range(S)]
    slot = max(t for _, t in jobs) * d
    slot_bytes = -(-slot // 16) * 16 + 4 * (-(-slot // 64))
    ring = P2PRing(rank, world, S, slot_bytes, gpu, dist, timeout_ms=30000)
    sched = RingSchedule(rank, world, S, len(jobs))
    st = _lib.stream_ptr(torch.cuda.current_stream())
    outs = []
    local = torch.empty(slot_bytes, dtype=torch.uint8, device=dev)
    for (j, t), x in zip(jobs, inputs):
        src, dst = sched.recv_from(j), sched.send_to(j)
        if src is not None:
            ring.wait(j, st)
        n = t * d
        y = torch.empty(t, d, device=dev)
        if rank == 0:
            base = ring.peer_slot(j)
            span.step_codes([seqs[j % S]], [t], in_f32=x, out_codes=DevPtr(base),
                            out_scales=DevPtr(base + -(-n // 16) * 16), out_f32=y)
        else:
            base = ring.local_slot(j)
            span.step_codes([seqs[j % S]], [t], in_codes=DevPtr(base), in_scales=DevPtr(base + -(-n // 16) * 16),
                            out_codes=local[:n].view(torch.int8), out_scales=local[-(-n // 16) * 16:][:4 * (-(-n // 64))].view(torch.float32),
                            out_f32=y)
            outs.append(y)
        if dst is not None:
            ring.signal(j if rank == 0 else j + S, st)
    torch.cuda.synchronize()
    if rank == 1:
        torch.save([o.cpu() for o in outs], "/tmp/p2p_rank1.pt")
    dist.barrier()
    if rank == 0:
        got = torch.load("/tmp/p2p_rank1.pt")
        a, b = make(0, 2), make(2, 4)
        sa = [a.new_sequence() for _ in range(S)]
        sb = [b.new_sequence() for _ in range(S)]
        bad = 0
        for k, ((j, t), x) in enumerate(zip(jobs, inputs)):
            n = t * d
            codes = torch.empty(n, dtype=torch.int8, device=dev)
            scales = torch.empty(-(-n // 64), device=dev)
            a.step_codes([sa[j % S]], [t], in_f32=x, out_codes=codes, out_scales=scales)
            y = torch.empty(t, d, device=dev)
            b.step_codes([sb[j % S]], [t], in_codes=codes, in_scales=scales, out_f32=y)
            same = torch.equal(y.cpu(), got[k])
            bad += 0 if same else 1
            print(f"job {j} t={t}: {'bit-identical' if same else 'MISMATCH'} "
                  f"(max |diff| {float((y.cpu() - got[k]).abs().max()):.3g})")
        print("P2P hop parity:", "OK" if bad == 0 else f"{bad} mismatches")
        if bad:
            sys.exit(1)
    ring.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
