"""Multi-GPU path on >= 2 GPUs: NCCL slab apply, slab dots/PCG and the slab V-cycle against the
single-GPU results and the oracle (tests/multi_gpu_worker.py under torchrun).

Skipped on fewer than 2 GPUs -- a skipped test has NOT passed: with one GPU the N > 1 path is
covered only by the one-GPU loopback tests (external-exchange mode) and tests/test_dist_gloo.py.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_nccl_slabs_vs_single_gpu_and_oracle(n):
    """n = 1 only self-checks the worker script on one GPU (one slab: no NCCL exchange runs)."""
    if gpus() < n:
        pytest.skip(f"needs {n} GPUs, found {gpus()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", str(n),
           os.path.join(ROOT, "tests", "multi_gpu_worker.py")] + (["--big"] if n >= 2 and n == min(8, gpus()) else [])
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"MULTI OK n={n}" in r.stdout


def test_peer_exchange_needs_nccl_slabs():
    """elas_set_peer_exchange is collective over an NCCL communicator: single-GPU and
    external-exchange ops are rejected with ELAS_EINVAL (runs on one GPU)."""
    if gpus() < 1:
        pytest.skip("no CUDA device")
    import synth
    from paper_2601_08374_b200 import elas
    from paper_2601_08374_b200.elas import Operator
    P = synth.make_problem("t", 2, 2, 4, 2, 4, seed=1)
    for kw in ({}, {"rank": 0, "nranks": 2}):
        op = Operator.from_problem(P, **kw)
        with pytest.raises(elas.ElasError, match="NCCL-mode"):
            op.set_peer_exchange(True)
        op.close()
