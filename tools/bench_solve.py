"""Time POBTAS / POBTASI on a C2-shaped factor."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib, perf
n, b, a = (int(x) for x in sys.argv[1:4])
lib = _lib.load(); dev = torch.device("cuda"); st = _lib.stream_ptr()
data = perf.device_random_spd_bta(n, b, a, seed=0)
ws = torch.empty(lib.stbta_pobtaf_workspace_bytes(n, b, a), dtype=torch.uint8, device=dev)
ld = torch.zeros(2, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.stbta_pobtaf(_lib.ptr(data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), ws.numel(), st)
torch.cuda.synchronize(); print("info", info.item())
N = n * b + a
x = torch.randn(N, dtype=torch.float64, device=dev)
wss = torch.empty(lib.stbta_pobtas_workspace_bytes(n, b, a, 1), dtype=torch.uint8, device=dev)
def ev(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(reps): fn()
    s1.record(); torch.cuda.synchronize(); return s0.elapsed_time(s1) / reps
for mode, name in ((1, "forward"), (2, "backward"), (0, "solve")):
    ms = ev(lambda: lib.stbta_pobtas(_lib.ptr(data), n, b, a, 1, _lib.ptr(x), 1, mode, _lib.ptr(wss), wss.numel(), st))
    print(f"pobtas {name}: {ms:.3f} ms  ({perf.bytes_pobtas(n,b,a)/(2 if mode else 1)/ms/1e6:.1f} GB/s of factor bytes)", flush=True)
prof = torch.zeros(24, dtype=torch.int64, device=dev)
lib.stbta_debug_set_profile(_lib.ptr(prof))
lib.stbta_pobtas(_lib.ptr(data), n, b, a, 1, _lib.ptr(x), 1, 1, _lib.ptr(wss), wss.numel(), st)
torch.cuda.synchronize(); lib.stbta_debug_set_profile(None)
p = prof.cpu().tolist(); c = max(p[20], 1)
print(f"fwd tiles {p[20]}: claim->pulled {p[21]/c/1e3:.2f} us, pulled->crit ready {p[22]/c/1e3:.2f} us, ready->publish {p[23]/c/1e3:.2f} us")
inv = torch.empty_like(data)
wsi = torch.empty(lib.stbta_pobtasi_workspace_bytes(n, b, a), dtype=torch.uint8, device=dev)
ms = ev(lambda: lib.stbta_pobtasi(_lib.ptr(data), _lib.ptr(inv), n, b, a, 1, _lib.ptr(wsi), wsi.numel(), st), reps=2)
print(f"pobtasi: {ms:.3f} ms  {perf.flops_pobtasi(n,b,a)/ms/1e9:.2f} TF/s", flush=True)
