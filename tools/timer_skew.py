"""%globaltimer offset and flag round-trip latency between SMs (CTA 0 vs every
other SM): does a cross-SM timeline (tools/prof_dag.py) need a skew correction?

    python tools/timer_skew.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_06938_b200 import _lib  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(_lib.__file__), "libstbta_tools.so"))
lib.stbta_debug_timer_skew.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
flags = torch.zeros(64 * sms, dtype=torch.int32, device="cuda")
out = torch.zeros(4 * sms, dtype=torch.int64, device="cuda")
rc = lib.stbta_debug_timer_skew(20, flags.data_ptr(), out.data_ptr(), None)
torch.cuda.synchronize()
assert rc == 0, rc
o = out.cpu().numpy().reshape(sms, 4)[1:].astype(np.float64)
rtt = (o[:, 2] - o[:, 0]) / 1e3
off = (o[:, 1] - (o[:, 0] + o[:, 2]) / 2) / 1e3
print(f"CTA 0 on SM {int(out[3].item())}; round trip us: min {rtt.min():.2f} median {np.median(rtt):.2f} max {rtt.max():.2f}")
print(f"clock offset of SM k vs SM of CTA 0 (us): min {off.min():.2f} median {np.median(off):.2f} max {off.max():.2f}")
for k in np.argsort(off)[:3].tolist() + np.argsort(off)[-3:].tolist():
    print(f"  sm {int(o[k, 3])}: offset {off[k]:.2f} us, rtt {rtt[k]:.2f} us")
