"""Time the UPDATE tile product in isolation for several CTA shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda"); st = _lib.stream_ptr()
for ntile in (148, 1024):
    A = torch.randn(ntile, 128, 128, dtype=torch.float64, device=dev)
    B = torch.randn(ntile, 128, 128, dtype=torch.float64, device=dev)
    C = torch.zeros(ntile, 128, 128, dtype=torch.float64, device=dev)
    for v in range(4):
        for grid in (148, 296):
            reps = 40
            rc = lib.stbta_debug_tile_bench(v, _lib.ptr(A), _lib.ptr(B), _lib.ptr(C), ntile, reps, grid, st)
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            rc = lib.stbta_debug_tile_bench(v, _lib.ptr(A), _lib.ptr(B), _lib.ptr(C), ntile, reps, grid, st)
            s1.record(); torch.cuda.synchronize()
            ms = s0.elapsed_time(s1)
            tiles = grid * reps
            print(f"ntile={ntile} variant={v} grid={grid} rc={rc}: {ms*1e3/reps:.1f} us/wave-rep  "
                  f"{2*128**3*tiles/ms/1e9:.2f} TF/s", flush=True)
