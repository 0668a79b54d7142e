"""Time the UPDATE tile product in isolation for several CTA shapes and depths."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib
lib = _lib.load_tools(); dev = torch.device("cuda"); st = _lib.stream_ptr()
ntile = 148
for K in (128, 256, 1024):
    A = torch.randn(ntile, 128, K, dtype=torch.float64, device=dev)
    B = torch.randn(ntile, 128, K, dtype=torch.float64, device=dev)
    C = torch.zeros(ntile, 128, 128, dtype=torch.float64, device=dev)
    for v in (3, 10, 11, 12):
        grid, reps = 148, max(4, 5120 // K)
        rc = lib.stbta_debug_tile_bench(v, _lib.ptr(A), _lib.ptr(B), _lib.ptr(C), ntile, reps, grid, K, st)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        rc = lib.stbta_debug_tile_bench(v, _lib.ptr(A), _lib.ptr(B), _lib.ptr(C), ntile, reps, grid, K, st)
        s1.record(); torch.cuda.synchronize()
        ms = s0.elapsed_time(s1)
        print(f"K={K} variant={v} rc={rc}: {ms*1e3/reps:.1f} us/tile  {2*128*128*K*grid*reps/ms/1e9:.2f} TF/s", flush=True)
out = torch.zeros(4, dtype=torch.float64, device=dev)
for mode in (0, 1, 2):
    for grid in (148, 296):
        iters = 2000
        lib.stbta_debug_lds_bench(mode, 10, grid, _lib.ptr(out), st); torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record(); lib.stbta_debug_lds_bench(mode, iters, grid, _lib.ptr(out), st); s1.record(); torch.cuda.synchronize()
        ms = s0.elapsed_time(s1)
        print(f"lds mode={mode} grid={grid}: {grid*8*iters*8*32*512/ms/1e9:.2f} TF/s", flush=True)
