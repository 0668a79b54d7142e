"""Does POBTAF overlap the chunked upload?  Device event timeline."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_06938_b200 import bta, perf, _lib

n, b, a = 48, 2048, 6
data = perf.device_random_spd_bta(n, b, a, seed=0)
host_in = data.cpu().pin_memory()
del data
torch.cuda.synchronize()
for rep in range(2):
    E = lambda: torch.cuda.Event(enable_timing=True)
    e0, e1, e2 = E(), E(), E()
    e0.record()
    m = bta.BTAMatrix(n, b, a, host_in)
    up_done = torch.cuda.Event(enable_timing=True)
    up_done.record(bta._side_stream(m._data.device, "upload"))
    e1.record()
    ld, info = bta.factorize_async(m, True)
    e2.record()
    torch.cuda.synchronize()
    print(f"upload {e0.elapsed_time(up_done):.1f} ms after e0; pobtaf launched at {e0.elapsed_time(e1):.1f}, "
          f"finished at {e0.elapsed_time(e2):.1f} ms; info={int(info.item())}; pipelined={m._upload is not None}", flush=True)
    # same without pipelining
    m2 = bta.BTAMatrix(n, b, a, host_in.cuda())
    torch.cuda.synchronize()
    e3, e4 = E(), E()
    e3.record(); bta.factorize_async(m2, True); e4.record(); torch.cuda.synchronize()
    print(f"plain pobtaf {e3.elapsed_time(e4):.1f} ms; equal={torch.equal(m._data, m2._data)}", flush=True)
# per-panel start times of the pipelined task graph (debug profile)
S = n * 16 + 1
prof = torch.zeros(64 + 12 * (S + 2), dtype=torch.int64, device="cuda")
lib = _lib.load()
m = bta.BTAMatrix(n, b, a, host_in)
lib.stbta_debug_set_profile(_lib.ptr(prof))
ld, info = bta.factorize_async(m, True)
torch.cuda.synchronize()
lib.stbta_debug_set_profile(None)
tl = prof[64:64 + 12 * (n * 16)].view(n * 16, 12).cpu().numpy().astype(np.float64) / 1e3
t0 = tl[0, 0]
print("panel POTRF deps-ok times (us from first claim):", [round(tl[s, 1] - t0) for s in range(0, n * 16, 64)])
print("panel POTRF end times:", [round(tl[s, 2] - t0) for s in range(0, n * 16, 64)])
# absolute: when does the task graph start relative to the upload?
gt = torch.zeros(4, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
lib.stbta_debug_globaltimer(_lib.ptr(gt[0:1]), _lib.stream_ptr(None))
m = bta.BTAMatrix(n, b, a, host_in)
up = bta._side_stream(m._data.device, "upload")
lib.stbta_debug_globaltimer(_lib.ptr(gt[1:2]), _lib.stream_ptr(None))
prof.zero_()
lib.stbta_debug_set_profile(_lib.ptr(prof))
ld, info = bta.factorize_async(m, True)
lib.stbta_debug_globaltimer(_lib.ptr(gt[2:3]), _lib.stream_ptr(None))
lib.stbta_debug_globaltimer(_lib.ptr(gt[3:4]), up.cuda_stream)
torch.cuda.synchronize()
lib.stbta_debug_set_profile(None)
g = gt.cpu().numpy().astype(np.float64) / 1e6
tl = prof[64:64 + 12 * (n * 16)].view(n * 16, 12).cpu().numpy().astype(np.float64) / 1e6
print(f"abs ms from t_ref: after BTAMatrix {g[1]-g[0]:.2f}, first worker claim {tl[0,0]-g[0]:.2f}, panel0 start {tl[0,1]-g[0]:.2f}, "
      f"panel 16*24 start {tl[16*24,1]-g[0]:.2f}, last panel end {tl[-1,2]-g[0]:.2f}, after pobtaf {g[2]-g[0]:.2f}, upload stream done {g[3]-g[0]:.2f}")
print("worker resident-wait (start, end) ms from t_ref per block:",
      [(round(tl[t*16,10]-g[0],2), round(tl[t*16,11]-g[0],2)) for t in range(0, 8)])
