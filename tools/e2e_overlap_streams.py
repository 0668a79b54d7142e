import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2507_06938_b200 import bta, perf
n, b, a = 48, 2048, 6
data = perf.device_random_spd_bta(n, b, a, seed=0)
host_in = data.cpu().pin_memory(); del data
torch.cuda.synchronize()
def run(tag):
    E = lambda: torch.cuda.Event(enable_timing=True)
    e0, e2 = E(), E()
    e0.record()
    m = bta.BTAMatrix(n, b, a, host_in)
    ld, info = bta.factorize_async(m, True)
    e2.record(); torch.cuda.synchronize()
    print(tag, f"upload+pobtaf {e0.elapsed_time(e2):.1f} ms", flush=True)
for _ in range(2): run("default stream:")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(2): run("pool stream:")
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if False else None
