"""End-to-end evaluate() with pageable numpy buffers vs pinned buffers (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5-hss"
spec, q = config(name)
inst = build_instance(spec)
ev = Evaluator(inst.cds)
n = inst.cds.n
w = np.asfortranarray(np.random.default_rng(1).standard_normal((n, q)))
y = np.empty((n, q), order="F")
ev.evaluate(w, out=y)
t = time.perf_counter()
for _ in range(3):
    ev.evaluate(w, out=y)
pageable = (time.perf_counter() - t) / 3
wh = torch.from_numpy(w.T.copy()).pin_memory()
yh = torch.empty_like(wh).pin_memory()
ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)
t = time.perf_counter()
for _ in range(3):
    ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)
pinned = (time.perf_counter() - t) / 3
same = bool(np.array_equal(y, yh.numpy().T))
print(f"{name}: pageable {pageable*1e3:.1f} ms, pinned {pinned*1e3:.1f} ms, same bits {same}")
