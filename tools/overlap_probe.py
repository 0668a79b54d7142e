"""Can a kernel on one stream overlap a pinned H2D copy on another (this box)?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib, bta
host = torch.empty(400_000_000, dtype=torch.float64).pin_memory()
dst = torch.empty_like(host, device="cuda")
x = torch.randn(8192, 8192, device="cuda", dtype=torch.float64)
up = torch.cuda.Stream()
def mm():
    for _ in range(6):
        y = x @ x
    return y
E = lambda: torch.cuda.Event(enable_timing=True)
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1, e2, e3 = E(), E(), E(), E()
    e0.record(); mm(); e1.record(); torch.cuda.synchronize()
    with torch.cuda.stream(up):
        e2.record(up); dst.copy_(host, non_blocking=True); e3.record(up)
    torch.cuda.synchronize()
    t_mm, t_cp = e0.elapsed_time(e1), e2.elapsed_time(e3)
    f0, f1 = E(), E()
    up.wait_stream(torch.cuda.current_stream())
    f0.record()
    with torch.cuda.stream(up):
        dst.copy_(host, non_blocking=True)
    mm()
    torch.cuda.current_stream().wait_stream(up)
    f1.record(); torch.cuda.synchronize()
    print(f"matmul {t_mm:.1f} ms, copy {t_cp:.1f} ms, both {f0.elapsed_time(f1):.1f} ms", flush=True)
# same with the library's chunked upload + memops
lib = _lib.load()
flags = torch.zeros(48, dtype=torch.int32, device="cuda")
n, b, a = 48, 2048, 6
host2 = host[: bta._storage_elems(n, b, a)]
dst2 = dst[: host2.numel()]
for rep in range(2):
    torch.cuda.synchronize(); flags.zero_(); torch.cuda.synchronize()
    f0, f1 = E(), E()
    f0.record()
    _lib.check(lib.stbta_upload_blocks(_lib.ptr(dst2), host2.data_ptr(), n, b, a, _lib.ptr(flags), 1, up.cuda_stream), "up")
    mm()
    torch.cuda.current_stream().wait_stream(up)
    f1.record(); torch.cuda.synchronize()
    print(f"chunked upload (memops) + matmul: {f0.elapsed_time(f1):.1f} ms", flush=True)
