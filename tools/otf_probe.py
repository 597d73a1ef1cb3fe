"""Near field on the fly vs resident (dev tool): device-resident evaluation time and resident
bytes of a BASELINE config built without D on the host (skip_near), uploaded with the near
field generated once (resident) and generated per evaluation (HMXG_UPLOAD_NEAR_ON_THE_FLY).
usage: python tools/otf_probe.py [cfg5-h2b] [q]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1812_07152_b200 import Evaluator, build_instance, config  # noqa: E402
from paper_1812_07152_b200.accuracy import Kernel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5-h2b"
spec, q = config(name)
if len(sys.argv) > 2:
    q = int(sys.argv[2])
spec.skip_near = True
t0 = time.time()
inst = build_instance(spec)
pts = inst.points()
kern = Kernel(spec.kernel, spec.h)
print(f"{name}: built in {time.time() - t0:.1f}s, |D| = {int(inst.cds.dptr[-1]) * 8 / 1e9:.2f} GB (not on the host)")
w = torch.randn(q, inst.cds.n, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
ys = {}
for otf in (False, True):
    t0 = time.time()
    ev = Evaluator(inst.cds, points=pts, kernel=kern, near_on_the_fly=otf)
    up = time.time() - t0
    y = torch.empty_like(w)
    for _ in range(2):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    torch.cuda.synchronize()
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=True, graph=False, sync=True)
    ph = ev.phases()
    gen_ms = sum(p["ms"] for p in ph if p["kind"] == "near-gen")
    leaf_ms = sum(p["ms"] for p in ph if p["kind"] == "near+leaf")
    waves = sum(1 for p in ph if p["kind"] == "near-gen")
    tf = inst.cds.flops(q) / (ms * 1e-3) / 1e12
    print(f"  {'on the fly' if otf else 'resident  '}: {ms:8.3f} ms  {tf:6.2f} TF/s (reference flop count)  "
          f"resident {ev.info().device_bytes / 1e9:6.2f} GB  upload {up:.1f}s  waves {waves}  gen {gen_ms:.3f} ms  "
          f"leaf waves {leaf_ms:.3f} ms", flush=True)
    ys[otf] = y.cpu()
    ev.close()
print(f"  bitwise equal: {torch.equal(ys[False], ys[True])}")
