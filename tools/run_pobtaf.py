"""One POBTAF on a random SPD BTA (for ncu captures): python tools/run_pobtaf.py n b a"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib, perf
n, b, a = (int(x) for x in sys.argv[1:4])
lib = _lib.load(); dev = torch.device("cuda"); st = _lib.stream_ptr()
data = perf.device_random_spd_bta(n, b, a, seed=0)
ws = torch.empty(lib.stbta_pobtaf_workspace_bytes(n, b, a), dtype=torch.uint8, device=dev)
ld = torch.zeros(2, dtype=torch.float64, device=dev); info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.stbta_pobtaf(_lib.ptr(data), n, b, a, 1, _lib.ptr(ld), _lib.ptr(info), _lib.ptr(ws), ws.numel(), st)
torch.cuda.synchronize(); print("info", info.item())
