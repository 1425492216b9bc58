"""CPU (gloo, world_size 2 and 3) tests of the span-to-span ring schedule
used by bench.py and the multi-GPU server: each rank adds its span's
contribution; the result of every session step must equal the sum over all
spans, sessions must not mix, and the schedule must not deadlock."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_01188_b200.pipeline import RingSchedule, run_jobs, split_blocks, torch_exchange


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sessions, steps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = sessions * steps
    sched = RingSchedule(rank, world, sessions, total)
    spans = split_blocks(10, world)
    start, end = spans[rank]
    done = []

    def step(j, payload):
        sess, k = j % sessions, j // sessions
        x = payload.clone() if payload is not None else torch.tensor([float(sess), 0.0])
        if rank == 0:
            x = torch.tensor([float(sess), x[1].item()])  # session id travels with the payload
        y = x.clone()
        y[1] += end - start  # "run" this span's blocks
        if rank == world - 1:
            done.append((sess, k, y[1].item()))
        return y

    run_jobs(sched, list(range(total)), step, torch_exchange, torch.empty(2))
    dist.barrier()
    dist.destroy_process_group()
    if rank == world - 1:
        q.put(done)


@pytest.mark.parametrize("world,sessions", [(2, 2), (3, 3), (2, 1)])
def test_ring_schedule_gloo(world, sessions):
    steps = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sessions, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    done = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every session step accumulated all 10 blocks once per step it went around the ring
    assert len(done) == sessions * steps
    for sess, k, val in done:
        assert val == 10.0 * (k + 1), (sess, k, val)
    assert sorted({s for s, _, _ in done}) == list(range(sessions))


def test_split_blocks():
    assert split_blocks(70, 8) == [(0, 9), (9, 18), (18, 27), (27, 36), (36, 45), (45, 54), (54, 62), (62, 70)]
    assert split_blocks(70, 1) == [(0, 70)]
    assert split_blocks(30, 2) == [(0, 15), (15, 30)]
