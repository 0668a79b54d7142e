"""Split-pair vs one-GPU f_obj throughput on 2 GPUs (C3): 8 points through
the gradient queue vs 8 sequential split-pair evaluations; asserts equal bits."""
import sys, time, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np, torch
from bench_inla import _c3_evaluator, TRI_THETA0
from paper_2507_06938_b200 import inla, sched
data, prior = _c3_evaluator()
evs = [inla.ObjectiveEvaluator(data.spec, prior=prior, device=torch.device("cuda", g)) for g in range(2)]
th = np.array(TRI_THETA0)
r = sched.GpuRunner(evs)
pts = [th + 1e-3 * k * np.ones(15) for k in range(1, 9)]
r.evaluate_points([th, th]); r.evaluate_points([th])
res = {}
for rep in range(2):
    inla.prior_cache_clear(); t0 = time.perf_counter()
    a = r._evaluate_queue(pts); res.setdefault("unsplit_8pts_s", []).append(time.perf_counter() - t0)
    inla.prior_cache_clear(); t0 = time.perf_counter()
    b = [r._evaluate_split([p])[0] for p in pts]; res.setdefault("split_8pts_s", []).append(time.perf_counter() - t0)
    assert a == b
    inla.prior_cache_clear(); t0 = time.perf_counter()
    evs[0].objective(th); res.setdefault("single_fobj_s", []).append(time.perf_counter() - t0)
print(json.dumps(res))
