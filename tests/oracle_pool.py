"""Parallel evaluation of oracle.apply_rows over chunks of rows (test infrastructure only).

The sampled-row oracle (oracle.apply_rows) evaluates each touched element stiffness row by
naive quadrature; thousands of rows at full size take minutes on one core.  This helper
splits the (sorted) rows into chunks and evaluates each chunk with oracle.apply_rows itself in
forked worker processes -- no arithmetic of its own: the result is the concatenation of the
oracle's answers.  Workers never touch CUDA.
"""

import multiprocessing as mp
import os

import numpy as np

import oracle

_STATE = {}


def _work(chunk):
    return oracle.apply_rows(_STATE["mesh"], _STATE["x"], chunk)


def apply_rows(mesh, x, rows, procs=None):
    rows = np.asarray(rows, dtype=np.int64).reshape(-1)
    procs = procs or min(os.cpu_count() or 1, 48)
    if procs <= 1 or rows.size < 256:
        return oracle.apply_rows(mesh, x, rows)
    order = np.argsort(rows, kind="stable")     # neighbouring rows share elements: keep them together
    chunks = [c for c in np.array_split(rows[order], procs * 4) if c.size]
    _STATE["mesh"], _STATE["x"] = mesh, x
    try:
        with mp.get_context("fork").Pool(procs) as pool:
            parts = pool.map(_work, chunks)
    finally:
        _STATE.clear()
    out = np.empty(rows.size)
    out[order] = np.concatenate(parts)
    return out
