"""First on-GPU check: DMMA peak, cuBLAS DGEMM, stbta_dgemm, POBTAF parity/timing."""
import ctypes, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
torch.cuda.init()
lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "paper_2507_06938_b200", "libstbta.so"))
vp = ctypes.c_void_p
dev = torch.device("cuda")
st = vp(torch.cuda.current_stream().cuda_stream)

def ev_time(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
    return best

print(torch.cuda.get_device_name(), flush=True)
scratch = torch.zeros(16, dtype=torch.float64, device=dev)
for blocks in (148, 296, 592):
    iters = 4000
    t = ev_time(lambda: lib.stbta_probe_dmma(blocks, iters, vp(scratch.data_ptr()), st))
    fl = blocks * 8 * iters * 16 * 512
    print(f"DMMA probe blocks={blocks}: {fl/t/1e12:.2f} TF/s", flush=True)

for N in (4096, 8192):
    A = torch.randn(N, N, dtype=torch.float64, device=dev); B = torch.randn(N, N, dtype=torch.float64, device=dev)
    t = ev_time(lambda: torch.matmul(A, B))
    print(f"torch DGEMM {N}: {2*N**3/t/1e12:.2f} TF/s", flush=True)
    C = torch.zeros(N, N, dtype=torch.float64, device=dev)
    lib.stbta_dgemm.argtypes = [ctypes.c_int]*5 + [ctypes.c_double, vp, ctypes.c_longlong, vp, ctypes.c_longlong, ctypes.c_double, vp, ctypes.c_longlong, vp]
    for ta, tb in ((0, 1), (0, 0), (1, 0)):
        f = lambda: lib.stbta_dgemm(ta, tb, N, N, N, 1.0, vp(A.data_ptr()), N, vp(B.data_ptr()), N, 0.0, vp(C.data_ptr()), N, st)
        t = ev_time(f)
        ref = (A.T if ta else A) @ (B.T if tb else B)
        err = ((C - ref).abs().max() / ref.abs().max()).item()
        print(f"stbta DGEMM ta={ta} tb={tb} {N}: {2*N**3/t/1e12:.2f} TF/s relerr {err:.2e}", flush=True)
    del A, B, C

from oracle import bta_np
lib.stbta_pobtaf_workspace_bytes.restype = ctypes.c_size_t
lib.stbta_pobtaf_workspace_bytes.argtypes = [ctypes.c_int]*3
lib.stbta_pobtaf.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, ctypes.c_size_t, vp]

def gpu_factor(data_np, n, b, a, use_arrow):
    d = torch.from_numpy(data_np).to(dev)
    ws_bytes = lib.stbta_pobtaf_workspace_bytes(n, b, a)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    ld = torch.zeros(1, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
    r = lib.stbta_pobtaf(vp(d.data_ptr()), n, b, a, use_arrow, vp(ld.data_ptr()), vp(info.data_ptr()), vp(ws.data_ptr()), ws_bytes, st)
    assert r == 0, r
    torch.cuda.synchronize()
    return d.cpu().numpy(), ld.item(), info.item()

rng = np.random.default_rng(0)
for (n, b, a) in [(1,1,0),(3,2,1),(5,3,2),(4,65,3),(6,130,2),(3,200,5),(4,257,70),(2,300,0)]:
    data = bta_np.random_spd_bta(rng, n, b, a)
    ref = data.copy(); ua = bta_np.factorize(ref, n, b, a)
    got, ld, info = gpu_factor(data, n, b, a, int(ua))
    err = np.abs(got - ref).max() / np.abs(ref).max()
    lref = bta_np.logdet(ref, n, b, a)
    print(f"pobtaf n={n} b={b} a={a}: maxrel {err:.2e} logdet {ld:.12e} ref {lref:.12e} rel {abs(ld-lref)/abs(lref):.2e} info {info}", flush=True)

# indefinite
data = bta_np.random_spd_bta(rng, 4, 70, 1); d,_,_,_ = bta_np.views(data, 4, 70, 1); d[2] = -np.eye(70)
_, _, info = gpu_factor(data, 4, 70, 1, 1); print("indefinite block 2 -> info", info)

# C2 timing: build SPD BTA on GPU from random L factor
n, b, a = 48, 2048, 6
N = bta_np.storage_elems(n, b, a)
g = torch.Generator(device=dev); g.manual_seed(0)
data = torch.empty(N, dtype=torch.float64, device=dev)
def make_c2():
    sd = 0.3 / b**0.5
    e0 = n*b*b; e1 = e0 + (n-1)*b*b; e2 = e1 + n*a*b
    D = data[:e0].view(n, b, b); Lo = data[e0:e1].view(n-1, b, b); Ar = data[e1:e2].view(n, a, b); T = data[e2:].view(a, a)
    torch.manual_seed(0)
    ld_ = torch.randn(n, b, b, dtype=torch.float64, device=dev) * sd
    ld_ = torch.tril(ld_, -1) + torch.diag_embed(1 + torch.rand(n, b, dtype=torch.float64, device=dev))
    ls = torch.randn(n-1, b, b, dtype=torch.float64, device=dev) * sd
    la = torch.randn(n, a, b, dtype=torch.float64, device=dev) * sd
    D.copy_(ld_ @ ld_.transpose(1, 2)); D[1:] += ls @ ls.transpose(1, 2)
    Lo.copy_(ls @ ld_[:-1].transpose(1, 2))
    Ar.copy_(la @ ld_.transpose(1, 2)); Ar[1:] += la[:-1] @ ls.transpose(1, 2)
    T.copy_(torch.eye(a, dtype=torch.float64, device=dev)*2 + (la @ la.transpose(1,2)).sum(0))
    del ld_, ls, la
make_c2(); torch.cuda.synchronize()
orig = data.clone()
ws_bytes = lib.stbta_pobtaf_workspace_bytes(n, b, a)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
ld = torch.zeros(1, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
for rep in range(3):
    data.copy_(orig); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    r = lib.stbta_pobtaf(vp(data.data_ptr()), n, b, a, 1, vp(ld.data_ptr()), vp(info.data_ptr()), vp(ws.data_ptr()), ws_bytes, st)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 1e3
    fl = bta_np.flops_pobtaf(n, b, a)
    print(f"C2 pobtaf: {t*1e3:.1f} ms  {fl/t/1e12:.2f} TF/s  logdet {ld.item():.10e} info {info.item()} r={r}", flush=True)
# check C2 logdet against torch cholesky of a few diag blocks? check via torch dense chol of first 2 blocks is costly; skip
