"""Per-step device time of one config with and without an L2 flush between steps (dev tool):
how much of a small problem's step is the cold start. usage: python tools/cold_probe.py [cfg1-hss]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1-hss"
spec, q = config(name)
inst = build_instance(spec)
ev = Evaluator(inst.cds)
w = torch.randn(q, inst.cds.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(w)
s = torch.cuda.Stream()
flush = torch.empty(int(256e6 // 4), dtype=torch.float32, device="cuda")
for mode in ("flush", "warm", "flush", "warm"):
    ts = []
    for it in range(30):
        with torch.cuda.stream(s):
            if mode == "flush":
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
            e1.record(s)
        e1.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{name} {mode:5s}: median {ts[len(ts) // 2]:.1f} us, min {ts[0]:.1f} us")
