"""The debug library (lib/libelas_debug.so, ELAS_DEBUG=1): every kernel family with device-side
bounds checks on, parity vs the oracle and zero failed checks (tests/debug_worker.py in a
subprocess, since the binding loads one library per process).  The stand-in for
compute-sanitizer, which is closed on this pool."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_library_bounds_checks():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = os.path.join(ROOT, "paper_2601_08374_b200", "lib", "libelas_debug.so")
    assert os.path.exists(lib), "build the debug library: python -m paper_2601_08374_b200.build --debug"
    env = dict(os.environ, ELAS_LIBNAME="libelas_debug.so")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "debug_worker.py")], capture_output=True,
                       text=True, timeout=1200, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "DEBUG OK" in r.stdout
