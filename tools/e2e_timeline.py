"""Host-side timeline of the e2e API sequence of bench.py (C2 by default)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_06938_b200 import bta, perf

n, b, a = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (48, 2048, 6)
data = perf.device_random_spd_bta(n, b, a, seed=0)
host_in = data.cpu().pin_memory()
del data
host_out = torch.empty(host_in.numel(), dtype=torch.float64).pin_memory()
rhs = np.random.default_rng(0).standard_normal(n * b + a)
torch.cuda.synchronize()

def step(sync_each):
    t = [time.perf_counter()]
    def mark():
        if sync_each:
            torch.cuda.synchronize()
        t.append(time.perf_counter())
    m = bta.BTAMatrix(n, b, a, host_in); mark()
    f = bta.factorize(m, use_arrow=True); mark()
    bta.logdet(f); mark()
    x = bta.solve(f, rhs); mark()
    s = bta.selected_invert(f, out=host_out); mark()
    s.numpy(out=host_out); mark()
    torch.cuda.synchronize(); mark()
    return np.diff(t) * 1e3

names = ["BTAMatrix", "factorize", "logdet", "solve", "selected_invert", "numpy(out)", "sync"]
for sync_each in (False, False, True):
    d = step(sync_each)
    print(("sync-each " if sync_each else "pipelined ") + " ".join(f"{k}={v:.1f}" for k, v in zip(names, d)) + f"  total={d.sum():.1f} ms", flush=True)
