"""Chunked bidirectional copy pipeline without the apply (the e2e upper bound of elas_apply_host):
64 z-chunks x 3 components, D2H of chunk k-1 concurrent with H2D of chunk k."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
N = 5467723800 // 8 // 3          # doubles per component (config 5)
h = torch.empty(3 * N, dtype=torch.float64).pin_memory()
h2 = torch.empty(3 * N, dtype=torch.float64).pin_memory()
d = torch.empty(3 * N, dtype=torch.float64, device="cuda")
d2 = torch.empty(3 * N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
import numpy as np
def ramp(nch, r):
    # chunk weights: the first and last chunks r times smaller than the middle ones
    w = np.ones(nch); w[0] = w[-1] = 1.0 / r
    if nch > 4: w[1] = w[-2] = 2.0 / r
    c = np.concatenate([[0], np.cumsum(w)]) / w.sum()
    return [int(N * x) for x in c]
for nch, r in ((32, 1), (64, 1), (32, 4), (64, 4), (32, 8), (48, 8)):
    bounds = ramp(nch, r)
    def run():
        evs = []
        for k in range(nch):
            with torch.cuda.stream(s1):
                for c in range(3):
                    a, b = c * N + bounds[k], c * N + bounds[k + 1]
                    d[a:b].copy_(h[a:b], non_blocking=True)
                ev = torch.cuda.Event(); ev.record(s1); evs.append(ev)
            if k > 0:
                with torch.cuda.stream(s2):
                    s2.wait_event(evs[k - 1])
                    for c in range(3):
                        a, b = c * N + bounds[k - 1], c * N + bounds[k]
                        h2[a:b].copy_(d2[a:b], non_blocking=True)
        with torch.cuda.stream(s2):
            s2.wait_event(evs[-1])
            for c in range(3):
                a, b = c * N + bounds[nch - 1], c * N + bounds[nch]
                h2[a:b].copy_(d2[a:b], non_blocking=True)
        torch.cuda.synchronize()
    run()
    t = time.perf_counter(); run(); dt = time.perf_counter() - t
    print(nch, "chunks, ramp", r, ":", round(dt * 1e3, 1), "ms ->", round(3 * N * 8 / dt / 1e9, 1), "GB/s per direction,",
          round(683465475 / dt / 1e9, 3), "GDoF/s equivalent")
