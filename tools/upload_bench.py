"""Upload time of a config with the near field shipped from the host vs generated on the
device, and the builder time saved by not forming D on the host (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config
from paper_1812_07152_b200.accuracy import Kernel

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5-h2b"
spec, q = config(name)
t = time.time(); full = build_instance(spec); tb_full = time.time() - t
spec.skip_near = True
t = time.time(); lean = build_instance(spec); tb_lean = time.time() - t
torch.cuda.synchronize()
t = time.time(); ev_s = Evaluator(full.cds); torch.cuda.synchronize(); tu_stored = time.time() - t
del ev_s
t = time.time(); ev_g = Evaluator(lean.cds, points=lean.points(), kernel=Kernel(spec.kernel, spec.h)); torch.cuda.synchronize()
tu_gen = time.time() - t
d_gb = full.cds.dptr[-1] * 8 / 1e9
print(f"{name}: |D| = {d_gb:.2f} GB; builder {tb_full:.1f} s with D, {tb_lean:.1f} s without; "
      f"upload {tu_stored:.2f} s shipping D, {tu_gen:.2f} s generating it on the device", flush=True)
w = np.asfortranarray(np.random.default_rng(0).standard_normal((full.cds.n, 64)))
from paper_1812_07152_b200.executor import Evaluator as E
y_g = ev_g.evaluate(w)
ev_s = E(full.cds)
y_s = ev_s.evaluate(w)
print(f"{name}: rel diff generated vs stored (64 columns) = {np.linalg.norm(y_g - y_s) / np.linalg.norm(y_s):.2e}")
