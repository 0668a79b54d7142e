import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bta_np
from paper_2507_06938_b200 import bta, bta_dist
for (n, b, a, P) in [(9, 20, 0, 2), (12, 20, 2, 3), (8, 20, 0, 2)]:
    rng = np.random.default_rng(1)
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy(); has = bta_np.factorize(ref, n, b, a)
    X = bta_np.selected_invert(ref, n, b, a, has)
    plan = bta_dist.plan_partitions(n, P)
    print("case", n, b, a, P, plan.boundaries, "seps", bta_dist._separators(plan), "ranges", bta_dist._partition_ranges(plan))
    f = bta_dist.d_factorize(bta.BTAMatrix(n, b, a, data), plan)
    G = bta_dist.d_selected_invert(f).numpy()
    d1, l1, a1, t1 = bta_np.views(G, n, b, a); d0, l0, a0, t0 = bta_np.views(X, n, b, a)
    print(" diag err", [f"{np.abs(d1[i]-d0[i]).max():.1e}" for i in range(n)])
    print(" lower err", [f"{np.abs(l1[i]-l0[i]).max():.1e}" for i in range(n-1)])
    if a: print(" arrow err", [f"{np.abs(a1[i]-a0[i]).max():.1e}" for i in range(n)], "tip", np.abs(t1-t0).max())
