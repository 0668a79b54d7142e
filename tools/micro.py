"""Microbenchmarks: DFMA vs DMMA rates, small GEMM latency, leaf kernel."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda"); st = _lib.stream_ptr()
lib.stbta_probe_dfma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / 1e3 / reps
sc = torch.zeros(4, dtype=torch.float64, device=dev)
for blocks in (1, 148, 592):
    it = 2000
    t = ev(lambda: lib.stbta_probe_dfma(blocks, it, _lib.ptr(sc), st))
    print(f"DFMA blocks={blocks}: {blocks*256*it*16/t/1e12:.3f} TF/s  ({t*1e6:.1f} us)", flush=True)
    t = ev(lambda: lib.stbta_probe_dmma(blocks, it, _lib.ptr(sc), st))
    print(f"DMMA blocks={blocks}: {blocks*8*it*16*512/t/1e12:.3f} TF/s  ({t*1e6:.1f} us)", flush=True)
t = ev(lambda: lib.stbta_probe_dmma(1, 1, _lib.ptr(sc), st), reps=50)
print(f"empty-ish launch: {t*1e6:.1f} us")
for (M, N, K) in [(64,64,64),(64,64,1024),(128,128,64),(2048,64,64),(2048,64,1024),(2048,2048,64),(2048,2048,2048),(1024,1024,1024)]:
    A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(N, K, dtype=torch.float64, device=dev)
    C = torch.zeros(M, N, dtype=torch.float64, device=dev)
    f = lambda: lib.stbta_dgemm(0, 1, M, N, K, 1.0, _lib.ptr(A), K, _lib.ptr(B), K, 0.0, _lib.ptr(C), N, st)
    t = ev(f, reps=20)
    tt = ev(lambda: torch.matmul(A, B.T), reps=20)
    print(f"gemm NT {M}x{N}x{K}: {t*1e6:8.1f} us {2*M*N*K/t/1e12:6.2f} TF/s | torch {tt*1e6:8.1f} us", flush=True)
