"""Run POBTAF on a small C2-shaped matrix (for ncu launch lists)."""
import ctypes, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib
n, b, a = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
lib = _lib.load()
dev = torch.device("cuda")
N = lib.stbta_storage_elems(n, b, a)
torch.manual_seed(0)
data = torch.zeros(N, dtype=torch.float64, device=dev)
e0 = n*b*b
D = data[:e0].view(n, b, b)
D.copy_(torch.eye(b, dtype=torch.float64, device=dev).expand(n, b, b) * 4.0)
e1 = e0 + (n-1)*b*b
data[e0:e1].uniform_(-1e-3, 1e-3)
e2 = e1 + n*a*b
data[e1:e2].uniform_(-1e-3, 1e-3)
data[e2:].view(a, a).copy_(torch.eye(a, dtype=torch.float64, device=dev) * 4.0)
orig = data.clone()
ws_bytes = lib.stbta_pobtaf_workspace_bytes(n, b, a)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
ld = torch.zeros(1, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
st = _lib.stream_ptr()
for r in range(reps):
    data.copy_(orig)
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    rc = lib.stbta_pobtaf(_lib.ptr(data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), ws_bytes, st)
    e.record(); torch.cuda.synchronize()
    print(f"rep {r}: {s.elapsed_time(e):.3f} ms rc={rc} info={info.item()} logdet={ld.item():.6f}", flush=True)
