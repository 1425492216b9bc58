"""Peer-memory hop (pb_hop.cu, pipeline.P2PRing) between two span processes:
the pipelined result must be bit-identical to handing the wire codes over in
one process (tools/p2p_check.py). Two GPUs: the mailbox is on the peer GPU
over NVLink. One GPU: both ranks share the device (same IPC mailbox and
signal/wait kernels, no NVLink)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_p2p_ring_bit_identical_to_single_process():
    import torch

    assert torch.cuda.device_count() >= 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "tools", "p2p_check.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "P2P hop parity: OK" in r.stdout, r.stdout[-3000:]
