"""Kernel-level breakdown of one C3 f_obj (device events around the phases via ncu-free timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_06938_b200 import inla
from tools.bench_inla import _c3_evaluator, TRI_THETA0
data, prior = _c3_evaluator()
ev = inla.ObjectiveEvaluator(data.spec, prior=prior)
th = np.array(TRI_THETA0)
ev.evaluate(th); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
inla.prior_cache_clear()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ev.evaluate(th); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
t0 = time.perf_counter()
for _ in range(3):
    inla.prior_cache_clear()
    ev.evaluate(th)
torch.cuda.synchronize()
print("f_obj s:", (time.perf_counter() - t0) / 3)
