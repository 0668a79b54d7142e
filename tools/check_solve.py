"""POBTAS / POBTASI parity vs the numpy oracle on small cases, plus C2-size timing."""
import ctypes, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_06938_b200 import _lib
from oracle import bta_np
lib = _lib.load(); dev = torch.device("cuda"); st = _lib.stream_ptr()
def fac(data, n, b, a, ua):
    d = torch.from_numpy(data).to(dev)
    wsb = lib.stbta_pobtaf_workspace_bytes(n, b, a); ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    ld = torch.zeros(1, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.check(lib.stbta_pobtaf(_lib.ptr(d), n, b, a, ua, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), wsb, st), "pobtaf")
    return d
def solve(d, n, b, a, ua, rhs, mode):
    x = torch.from_numpy(np.ascontiguousarray(rhs)).to(dev)
    nr = 1 if rhs.ndim == 1 else rhs.shape[1]
    wsb = lib.stbta_pobtas_workspace_bytes(n, b, a, nr); ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.check(lib.stbta_pobtas(_lib.ptr(d), n, b, a, ua, _lib.ptr(x), nr, mode, _lib.ptr(ws), wsb, st), "pobtas")
    torch.cuda.synchronize(); return x.cpu().numpy()
def selinv(d, n, b, a, ua):
    inv = torch.empty_like(d)
    wsb = lib.stbta_pobtasi_workspace_bytes(n, b, a); ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    _lib.check(lib.stbta_pobtasi(_lib.ptr(d), _lib.ptr(inv), n, b, a, ua, _lib.ptr(ws), wsb, st), "pobtasi")
    torch.cuda.synchronize(); return inv.cpu().numpy()
rng = np.random.default_rng(7)
worst = {"fwd":0, "bwd":0, "solve":0, "sinv":0}
for (n, b, a, nr) in [(1,1,0,1),(3,2,1,1),(5,3,2,2),(4,65,3,1),(6,130,2,3),(3,200,5,9),(4,257,7,1),(2,300,0,1),(8,64,1,1),(2,5,4,1)]:
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy(); ua = bta_np.factorize(ref, n, b, a)
    d = fac(data, n, b, a, int(ua))
    N = n*b+a
    rhs = rng.normal(size=(N,) if nr == 1 else (N, nr))
    for mode, name, fn in ((1, "fwd", bta_np.forward), (2, "bwd", bta_np.backward), (0, "solve", bta_np.solve)):
        got = solve(d, n, b, a, int(ua), rhs, mode)
        exp = fn(ref, n, b, a, ua, rhs)
        err = np.abs(got - exp).max() / np.abs(exp).max()
        worst[name] = max(worst[name], err)
    gi = selinv(d, n, b, a, int(ua)); ei = bta_np.selected_invert(ref, n, b, a, ua)
    err = np.abs(gi - ei).max() / np.abs(ei).max(); worst["sinv"] = max(worst["sinv"], err)
    print(n, b, a, nr, {k: f"{v:.1e}" for k, v in worst.items()}, flush=True)
# timing at C2 shape (diagonally dominant synthetic)
n, b, a = 48, 2048, 6
N = lib.stbta_storage_elems(n, b, a)
data = torch.zeros(N, dtype=torch.float64, device=dev); e0 = n*b*b
data[:e0].view(n, b, b).copy_(torch.eye(b, dtype=torch.float64, device=dev).expand(n, b, b) * 4.0)
e1 = e0 + (n-1)*b*b; data[e0:e1].uniform_(-1e-3, 1e-3); e2 = e1 + n*a*b; data[e1:e2].uniform_(-1e-3, 1e-3)
data[e2:].view(a, a).copy_(torch.eye(a, dtype=torch.float64, device=dev) * 4.0)
wsb = lib.stbta_pobtaf_workspace_bytes(n, b, a); ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
ld = torch.zeros(1, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.stbta_pobtaf(_lib.ptr(data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), wsb, st)
x = torch.randn(n*b+a, dtype=torch.float64, device=dev)
wsb2 = lib.stbta_pobtas_workspace_bytes(n, b, a, 1); ws2 = torch.empty(wsb2, dtype=torch.uint8, device=dev)
for r in range(3):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); lib.stbta_pobtas(_lib.ptr(data), n, b, a, 1, _lib.ptr(x), 1, 0, _lib.ptr(ws2), wsb2, st); e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e)/1e3
    print(f"C2 pobtas: {t*1e3:.2f} ms  {bta_np.bytes_pobtas(n,b,a)/t/1e9:.0f} GB/s", flush=True)
inv = torch.empty_like(data)
wsb3 = lib.stbta_pobtasi_workspace_bytes(n, b, a); ws3 = torch.empty(wsb3, dtype=torch.uint8, device=dev)
for r in range(2):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); rc = lib.stbta_pobtasi(_lib.ptr(data), _lib.ptr(inv), n, b, a, 1, _lib.ptr(ws3), wsb3, st); e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e)/1e3
    print(f"C2 pobtasi: {t*1e3:.1f} ms  {bta_np.flops_pobtasi(n,b,a)/t/1e12:.2f} TF/s rc={rc}", flush=True)
