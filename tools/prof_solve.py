"""POBTAS sweep timing breakdown (device %globaltimer per tile through the
stbta_debug_set_profile hook): per tile, time spent folding the pulled
dependencies, waiting for / loading the pushed neighbour product, and the
critical step (W gemv, push gemv, publish).

    python tools/prof_solve.py n b a
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_06938_b200 import _lib, bta, perf  # noqa: E402

n, b, a = (int(x) for x in sys.argv[1:4])
lib = _lib.load()
dev = torch.device("cuda")
m = bta.BTAMatrix(n, b, a, perf.device_random_spd_bta(n, b, a, seed=0))
f = bta.factorize(m, use_arrow=True)
x0 = torch.randn(m.dim, dtype=torch.float64, device=dev)
for mode, name in ((1, "forward"), (2, "backward"), (0, "solve")):
    x = x0.clone()
    bta._pobtas(f, x, mode)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x = x0.clone()
    s0.record()
    bta._pobtas(f, x, mode)
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1)
    nb = perf.bytes_pobtas(n, b, a) / (2 if mode else 1)
    print(f"{name}: {ms:.3f} ms, {nb / ms / 1e6:.1f} GB/s of factor bytes")
prof = torch.zeros(64, dtype=torch.int64, device=dev)
lib.stbta_debug_set_profile(_lib.ptr(prof))
x = x0.clone()
bta._pobtas(f, x, 1)
torch.cuda.synchronize()
lib.stbta_debug_set_profile(None)
p = prof.cpu().tolist()
c = max(p[20], 1)
print(f"forward sweep, {p[20]} tiles: pulled folds {p[21] / c / 1e3:.2f} us/tile, "
      f"push load + neighbour wait {p[22] / c / 1e3:.2f} us/tile, "
      f"critical step {p[23] / c / 1e3:.2f} us/tile")
