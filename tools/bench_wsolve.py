"""Tile-sweep POBTAS vs the W-based POBTAS (block inverses shared with
POBTASI) at one BTA shape: device times of each piece, and the agreement of
the two solves.

    python tools/bench_wsolve.py n b a [nrhs]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_06938_b200 import bta, perf  # noqa: E402

n, b, a = (int(x) for x in sys.argv[1:4])
nrhs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device("cuda")
m = bta.BTAMatrix(n, b, a, perf.device_random_spd_bta(n, b, a, seed=0))
f = bta.factorize(m, use_arrow=True)
x0 = torch.randn(m.dim, nrhs, dtype=torch.float64, device=dev).squeeze(1)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        fn()
        s1.record()
        torch.cuda.synchronize()
        out.append(s0.elapsed_time(s1))
    return min(out), sorted(out)[len(out) // 2]


quick = os.environ.get("BW_QUICK") == "1"  # W solve only (parameter sweeps)
res = {"n": n, "b": b, "a": a, "nrhs": nrhs,
       "chunk": os.environ.get("STBTA_WS_CHUNK"), "colmap": os.environ.get("STBTA_WS_COLMAP"), "u": os.environ.get("STBTA_WS_U")}
for mode, name in ((1, "forward"), (2, "backward"), (0, "solve")):
    if not quick:
        res[f"tile_{name}_ms"] = timed(lambda: bta._pobtas(f, x0.clone(), mode, policy="tile"))


def prep():
    f._si_ws = None
    bta.prepare_inverse(f)


res["prepare_ms"] = timed(prep)
for mode, name in ((1, "forward"), (2, "backward"), (0, "solve")):
    res[f"w_{name}_ms"] = timed(lambda: bta._pobtas(f, x0.clone(), mode, policy="w"))
if not quick:
    si = f._si_ws
    f._si_ws = None
    res["selinv_plain_ms"] = timed(lambda: bta.selected_invert(f), reps=3)
    f._si_ws = si
    res["selinv_prepared_ms"] = timed(lambda: bta.selected_invert(f), reps=3)
xt = x0.clone()
bta._pobtas(f, xt, 0, policy="tile")
xw = x0.clone()
bta._pobtas(f, xw, 0, policy="w")
res["max_rel_diff"] = float(((xw - xt).abs().max() / xt.abs().max()).item())
if os.environ.get("BW_PROF") == "1":  # per-phase device time (CTA 0, %globaltimer)
    from paper_2507_06938_b200 import _lib

    lib = _lib.load()
    prof = torch.zeros(64, dtype=torch.int64, device=dev)
    lib.stbta_debug_set_profile(_lib.ptr(prof))
    bta._pobtas(f, x0.clone(), 0, policy="w")
    torch.cuda.synchronize()
    lib.stbta_debug_set_profile(None)
    ph = prof.cpu().tolist()[40:49]
    names = ["f_L", "f_W", "f_arrow", "f_tip", "b_tip", "b_LT", "b_z", "b_WT", "b_red"]
    res["phase_us"] = {k: v / 1e3 for k, v in zip(names, ph)}
gb = perf.bytes_pobtas(n, b, a) / 1e9
res["solve_factor_GB"] = gb
print(json.dumps(res))
