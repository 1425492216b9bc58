"""CPU (gloo, world size 2) test of the box front end's control plane
(paper_2209_01188_b200.box): rank 0's BoxScheduler coalesces concurrent
STEPs, splits a long prompt into causal chunk jobs, reserves pages and sends
one descriptor per job; rank 1 (serve_rank) must apply the identical job
sequence with identical per-sequence positions and page counts, so its KV
pool mirrors rank 0's. The GPU data path (sub-span step, mailbox hop,
egress) is replaced by a recording fake; the GPU tests cover it."""

import os
import socket
import threading

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_01188_b200.box import OP_STOP, BoxPlan, BoxScheduler, BoxSequence, RankState, serve_rank
from paper_2209_01188_b200.model import ModelConfig
from paper_2209_01188_b200.server import ServerConfig
from paper_2209_01188_b200.span import PagePool

D = 8


class FakeSpan:
    def __init__(self, pages, page_tokens):
        self.pool = PagePool(pages)
        self.page_tokens = page_tokens
        self.device = torch.device("cpu")
        self.n_blocks = 2
        self.config = ModelConfig(4, D, 2, 32, 64)

    def pages_needed(self, seq, new_len):
        return max(0, -(-new_len // self.page_tokens) - len(seq.pages))

    def reserve(self, seq, new_len):
        need = self.pages_needed(seq, new_len)
        if need:
            seq.pages.extend(self.pool.alloc(need))

    def release(self, seq):
        self.pool.free(seq.pages)
        seq.pages = []
        seq.length = 0


class _Done:
    def synchronize(self):
        pass


class FakeRank(RankState):
    """Records every hop (job id, per-sequence lengths before the step, new
    positions, free pages after the reservation); rank 0's 'ring' returns x + 1."""

    def __init__(self, plan, rank, span):
        super().__init__(plan, rank, span, ring=None, dist=dist)
        self.log, self.outs = [], {}

    def bind_thread(self):
        pass

    def new_stream(self):
        return None

    def finish(self):
        pass

    def close(self):
        pass

    def hop(self, j, seqs, lens, x=None, tape=None):
        self.log.append((j, [s.length for s in seqs], list(lens), self.span.pool.free_pages))
        for s, t in zip(seqs, lens):
            s.length += t
        if self.rank == 0:
            self.outs[j] = x + 1

    def egress(self, j, n_tok, stream):
        return _Done(), self.outs.pop(j)


def _plan():
    cfg = ServerConfig(seed=1, model=ModelConfig(4, D, 2, 32, 64), capacity=4, max_batch_tokens=4, page_tokens=2,
                       cache_budget_tokens=64, blocks=(0, 4))
    return BoxPlan(cfg, 2)


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    plan = _plan()
    span = FakeSpan(plan.pages(4), plan.config.page_tokens)
    st = FakeRank(plan, rank, span)
    if rank == 1:
        serve_rank(plan, 1, dist, state=st)
        q.put(("rank1", st.log))
    else:
        sch = BoxScheduler(st, plan)
        seqs = [BoxSequence() for _ in range(3)]
        results = {}
        # a 9-token prompt (> max_batch_tokens 4: chunks 4, 4, 1), then concurrent decode steps
        x = torch.arange(9 * D, dtype=torch.float32).view(9, D)
        results["long"] = sch.run(seqs[0], x)

        def decode(i):
            results[i] = [sch.run(seqs[i], torch.full((1, D), float(i * 10 + k))) for k in range(5)]

        ts = [threading.Thread(target=decode, args=(i,)) for i in range(3)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        sch.call("release", seqs[1])
        sch.run(seqs[2], torch.zeros(3, D))
        sch.stop()
        # plain Python / numpy only: tensors would travel as shared-memory handles
        # that vanish when this process exits before the parent reads them
        results = {k: (v.numpy() if torch.is_tensor(v) else [r.numpy() for r in v]) for k, v in results.items()}
        q.put(("rank0", (st.log, results, sch.batches, sch.batched_steps, span.pool.free_pages)))
    dist.destroy_process_group()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_box_control_plane_mirrors_rank0():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=100) for _ in range(2))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    log0, results, batches, batched, free0 = got["rank0"]
    log1 = got["rank1"]
    # identical job stream on both ranks: same job ids, same per-sequence positions and lengths
    assert [(j, L, t) for j, L, t, _ in log0] == [(j, L, t) for j, L, t, _ in log1]
    # rank 1 reserves lazily, never more than rank 0 (which reserved the long prompt up front)
    assert all(f1 >= f0 for (*_, f0), (*_, f1) in zip(log0, log1))
    # the long prompt ran as causal chunks 4 + 4 + 1 on sequence 0
    assert [(L, t) for _, L, t, _ in log0[:3]] == [([0], [4]), ([4], [4]), ([8], [1])]
    assert (results["long"] == torch.arange(9 * D, dtype=torch.float32).view(9, D).numpy() + 1).all()
    for i in range(3):
        assert [float(r[0, 0]) for r in results[i]] == [i * 10 + k + 1.0 for k in range(5)]
    # concurrent decode steps of distinct sessions were coalesced into shared jobs
    assert batched == 3 * 5 + 3 + 1 and batches < batched
    assert OP_STOP == 6
