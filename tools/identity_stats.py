"""Executed vs algorithmic flops of the lowered plan (identity rows of the bases, dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

for name in sys.argv[1:] or ["cfg1-hss", "cfg5-hss"]:
    spec, q = config(name)
    inst = build_instance(spec)
    ev = Evaluator(inst.cds)
    w = torch.randn(q, inst.cds.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    s = torch.cuda.Stream()
    ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=True, graph=False, levels=True)
    torch.cuda.synchronize()
    ph = ev.phases()
    ex = sum(p["flops_per_col"] for p in ph) * q
    alg = inst.cds.flops(q)
    print(f"{name}: executed {ex:.3e} algorithmic {alg:.3e} ratio {ex/alg:.3f}")
    for p in ph:
        if p["kind"] in ("gather", "scatter"):
            continue
        print(f"   {p['kind']:14s} L{p['level']:<3d} {p['ms']:.4f} ms  {p['flops_per_col']*q/max(p['ms'],1e-9)/1e9:.2f} TF/s  "
              f"tiles={p['tiles']}")
