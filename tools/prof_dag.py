"""POBTAF task-graph timing breakdown (device globaltimer per task kind)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib, perf
n, b, a = (int(x) for x in sys.argv[1:4])
lib = _lib.load()
dev = torch.device("cuda")
data0 = perf.device_random_spd_bta(n, b, a, seed=0)
data = data0.clone()
ws = torch.empty(lib.stbta_pobtaf_workspace_bytes(n, b, a), dtype=torch.uint8, device=dev)
ld = torch.zeros(2, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
prof = torch.zeros(18, dtype=torch.int64, device=dev)
st = _lib.stream_ptr()
def run():
    data.copy_(data0)
    return lib.stbta_pobtaf(_lib.ptr(data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), ws.numel(), st)
run(); torch.cuda.synchronize()
for r in range(2):
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    data.copy_(data0); s0.record()
    lib.stbta_pobtaf(_lib.ptr(data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), ws.numel(), st)
    s1.record(); torch.cuda.synchronize()
    ms = s0.elapsed_time(s1)
    print(f"pobtaf {n}x{b}x{a}: {ms:.3f} ms  {perf.flops_pobtaf(n,b,a)/ms/1e9:.2f} TF/s info={info.item()}", flush=True)
lib.stbta_debug_set_profile(_lib.ptr(prof))
run(); torch.cuda.synchronize()
lib.stbta_debug_set_profile(None)
p = prof.cpu().tolist()
for k, name in enumerate(["POTRF", "TRSM", "UPDATE", "STRIP"]):
    c, w, e = p[3*k:3*k+3]
    if c:
        print(f"{name:7s} n={c:8d} wait {w/c/1e3:9.2f} us/task exec {e/c/1e3:9.2f} us/task  total exec {e/1e6:9.2f} ms wait {w/1e6:9.2f} ms")
print("POTRF phases (us per task): A %.2f C %.2f - %.2f - %.2f store %.2f load %.2f" % tuple(x/1e3/max(p[0],1) for x in p[12:18]))
