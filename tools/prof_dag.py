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
prof = torch.zeros(64 + 12 * (n * ((b + 127) // 128) + (a + 127) // 128 + 2), dtype=torch.int64, device=dev)
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
c = max(p[3], 1); cs = max(p[9], 1)
print("TRSM: wait->loaded %.2f us, trsm_strip_smem %.2f us, store+signal %.2f us" % (p[18]/c/1e3, p[19]/c/1e3, (p[5]-p[18]-p[19])/c/1e3))
print("STRIP: load+mma %.2f us, store+signal %.2f us" % (p[20]/cs/1e3, (p[11]-p[20])/cs/1e3))
cu = max(p[6], 1)
print("UPDATE: C load + tile_mma %.2f us, store+signal %.2f us" % (p[22]/cu/1e3, (p[8]-p[22])/cu/1e3))
import numpy as np
S = n * ((b + 127) // 128)
tl = np.array(p[64:64 + 12 * S], dtype=np.int64).reshape(S, 12).astype(np.float64) / 1e3
rng = range(1, S - 1)
def avg(f): return np.mean([f(s) for s in rng])
print("critical chain per panel (us): potrf exec %.2f | potrf_end -> trsm deps ok %.2f | trsm exec %.2f | trsm_end -> strip deps ok %.2f | strip exec %.2f | strip_end -> next potrf deps ok %.2f" % (
    avg(lambda s: tl[s,2]-tl[s,1]), avg(lambda s: tl[s,4]-tl[s,2]), avg(lambda s: tl[s,5]-tl[s,4]),
    avg(lambda s: tl[s,7]-tl[s,5]), avg(lambda s: tl[s,8]-tl[s,7]), avg(lambda s: tl[s+1,1]-tl[s,8])))
print("claims: trsm claimed %.2f us before potrf end, strip claimed %.2f us before trsm end; G1 strip end - potrf_end(s) %.2f us; next potrf t1 - g1 end %.2f" % (
    avg(lambda s: tl[s,2]-tl[s,3]), avg(lambda s: tl[s,5]-tl[s,6]), avg(lambda s: tl[s,9]-tl[s,2]), avg(lambda s: tl[s+1,1]-tl[s,9])))
print("panel period %.2f us" % avg(lambda s: tl[s+1,2]-tl[s,2]))
print("tile (s+1,s) last prior update: claimed %.2f us, done %.2f us relative to POTRF(s) end" % (
    avg(lambda s: tl[s,10]-tl[s,2]), avg(lambda s: tl[s,11]-tl[s,2])))
