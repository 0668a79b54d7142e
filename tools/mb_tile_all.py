import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2507_06938_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda"); st = _lib.stream_ptr()
ntile = 148
for K in (128, 1024):
    A = torch.randn(ntile, 128, K, dtype=torch.float64, device=dev)
    B = torch.randn(ntile, 128, K, dtype=torch.float64, device=dev)
    C = torch.zeros(ntile, 128, 128, dtype=torch.float64, device=dev)
    for v in range(13):
        grid, reps = 148, max(4, 5120 // K)
        rc = lib.stbta_debug_tile_bench(v, _lib.ptr(A), _lib.ptr(B), _lib.ptr(C), ntile, reps, grid, K, st)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        rc = lib.stbta_debug_tile_bench(v, _lib.ptr(A), _lib.ptr(B), _lib.ptr(C), ntile, reps, grid, K, st)
        s1.record(); torch.cuda.synchronize()
        ms = s0.elapsed_time(s1)
        print(f"K={K} variant={v} rc={rc}: {ms*1e3/reps:.1f} us/tile  {2*128*128*K*grid*reps/ms/1e9:.2f} TF/s", flush=True)
