"""Multi-GPU parity: the octree domain decomposition over NCCL reproduces the
single-GPU matvec (also with the curvature self-term), GMRES solve and BIBEE energy, and the
host-buffer product equals the device one.  Needs >= 2 GPUs (skipped otherwise)."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("case", ["lyso40", "c3"])
def test_two_gpus_match_one(case):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + (os.getpid() % 200)),
           os.path.join(ROOT, "tools", "mgpu_check.py"), case]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    line = [l for l in out.stdout.splitlines() if l.startswith("MGPU ")]
    assert line, out.stdout[-2000:] + out.stderr[-2000:]
    r = json.loads(line[0][5:])
    assert r["matvec_rel"] < 1e-6
    assert r["self_term_rel"] < 1e-6  # option self_term = 1 on the domain decomposition
    assert r["host_rel"] == 0.0  # host-buffer product = device product (same path on N > 1)
    g, o, gi, oi = r["solve"]
    assert abs(g / o - 1) < 1e-6 and abs(gi - oi) <= 1
    assert abs(r["bibee"][0] / r["bibee"][1] - 1) < 1e-6
    assert min(r["n_local"]) > 0
