"""One C2 step (POBTAF + W pass + POBTAS on W + POBTASI on the n=48, b=2048, a=6 matrix,
as bench.py times it) for ncu captures:

    ncu --set full --clock-control none -k regex:sinv_persistent -c 1 -o rep python tools/run_c2_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_06938_b200 import bta, perf  # noqa: E402

n, b, a = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (48, 2048, 6)))
m = bta.BTAMatrix(n, b, a, perf.device_random_spd_bta(n, b, a, seed=1234))
f = bta.factorize(m, use_arrow=True)
if os.environ.get("STBTA_SOLVE", "auto") != "tile":
    bta.prepare_inverse(f)  # W shared by the solve and the selected inversion (bench.py --solve w)
x = bta.solve(f, torch.ones(m.dim, dtype=torch.float64, device=m.device))
inv = bta.selected_invert(f)
torch.cuda.synchronize()
print("logdet", bta.logdet(f))
