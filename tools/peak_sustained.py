"""Sustained FP64 DMMA / DFMA peak with clocks sampled during the run."""
import sys, os, subprocess, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2507_06938_b200 import _lib
lib = _lib.load_tools(); dev = torch.device("cuda"); st = _lib.stream_ptr()
sc = torch.zeros(16, dtype=torch.float64, device=dev)
for name, fn, fl in (("dmma", _lib.load().stbta_probe_dmma, lambda b, it: b * 8 * it * 16 * 512),
                     ("dfma", lib.stbta_probe_dfma, lambda b, it: b * 256 * it * 16)):
    blocks, iters = 148 * 4, 20000
    fn(blocks, 100, _lib.ptr(sc), st); torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
    s0.record()
    reps = 0
    t0 = time.time()
    while time.time() - t0 < 3.0:
        fn(blocks, iters, _lib.ptr(sc), st); reps += 1
        if reps % 4 == 0: torch.cuda.synchronize()
    s1.record(); torch.cuda.synchronize()
    p.terminate(); out = p.communicate()[0]
    clk = [float(l.split(",")[0]) for l in out.strip().splitlines() if l.strip()]
    pw = [float(l.split(",")[1]) for l in out.strip().splitlines() if l.strip()]
    ms = s0.elapsed_time(s1)
    print(f"{name} sustained: {fl(blocks, iters) * reps / ms / 1e9:.2f} TF/s over {ms:.0f} ms; "
          f"sm clock median {statistics.median(clk):.0f} MHz min {min(clk):.0f}; power max {max(pw):.0f} W; reasons {set(l.split(',')[2].strip() for l in out.strip().splitlines())}", flush=True)
