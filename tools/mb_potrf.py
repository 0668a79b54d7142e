"""Time the in-CTA 128x128 Cholesky + inverse in isolation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib
lib = _lib.load_tools(); dev = torch.device("cuda"); st = _lib.stream_ptr()
X = torch.randn(128, 128, dtype=torch.float64, device=dev) * 0.05
A = (X @ X.T + torch.eye(128, dtype=torch.float64, device=dev) * 2).contiguous()
out = torch.zeros(4, dtype=torch.float64, device=dev)
ph = torch.zeros(6, dtype=torch.int64, device=dev)
ref = torch.linalg.cholesky(A)
for grid in (1, 148):
    reps = 50
    lib.stbta_debug_potrf_bench(_lib.ptr(A), _lib.ptr(out), reps, grid, _lib.ptr(ph), st)
    torch.cuda.synchronize()
    p = ph.cpu().tolist()
    print(f"grid={grid}: {p[5]/reps/1e3:.2f} us/potrf  phases us: A(tall factor|upd) {p[0]/reps/1e3:.2f} C(next column) {p[1]/reps/1e3:.2f} "
          f"logdet {out[0].item():.12f} ref {2*torch.log(torch.diagonal(ref)).sum().item()/2:.12f}"
          f" W[127,0] {out[1].item():.6e} ref {torch.linalg.inv(ref)[127,0].item():.6e}", flush=True)
cyc = torch.zeros(1, dtype=torch.int64, device=dev)
for which, name in ((0, "DMMA"), (1, "DFMA")):
    for it in (64, 1024):
        lib.stbta_debug_latency(which, it, _lib.ptr(out), _lib.ptr(cyc), st); torch.cuda.synchronize()
        print(f"{name} dependent chain: {cyc.item()/it:.1f} clk per op (iters={it})")
