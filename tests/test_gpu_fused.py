"""The fused-operand decode GEMV (operand warps build the int8-digit B
fragments in shared memory) must produce bit-identical hidden states to the
k_fragwrite path, with outlier features present, at the 560M and the 176B
shapes (tools/fused_check.py with and without BlockSpan(operand_kernel=True))."""

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_fused_operand_bit_identical_to_fragwrite(tmp_path):
    outs = []
    for fused in (True, False):
        f = tmp_path / f"out_{int(fused)}.npy"
        args = [sys.executable, os.path.join(ROOT, "tools", "fused_check.py"), str(f)] + ([] if fused else ["kernel"])
        r = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
        outs.append(np.load(f))
        assert "outliers per matrix" in r.stdout
    assert outs[0].shape == outs[1].shape
    assert np.isfinite(outs[0]).all()
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
