"""End-to-end (host buffers) time per pipeline chunk width (dev tool; HMXG_CHUNK_COLS)."""
import os, subprocess, sys
for cfg in sys.argv[1:] or ["cfg2-h2b", "cfg3-h2b"]:
    for cc in (64, 128, 256, 512):
        env = dict(os.environ, HMXG_CHUNK_COLS=str(cc))
        out = subprocess.run([sys.executable, "-c", f"""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_1812_07152_b200 import Evaluator, build_instance, config
spec, q = config('{cfg}'); inst = build_instance(spec); ev = Evaluator(inst.cds)
wh = torch.randn((q, inst.cds.n), dtype=torch.float64).pin_memory(); yh = torch.empty_like(wh).pin_memory()
for _ in range(2): ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)
t = time.perf_counter()
for _ in range(5): ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)
dt = (time.perf_counter() - t) / 5
print(f'{cfg} chunk={cc}: {{dt*1e3:.2f}} ms {{inst.cds.flops(q)/dt/1e12:.2f}} TF/s')
"""], env=env, capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-300:], flush=True)
