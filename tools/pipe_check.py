"""Subtree-pipelined claim order (HMXG_PIPE) against the level-major order: same bits, and the
device-resident time of each (dev tool). Usage: pipe_check.py CFG[:Q] [d0 ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

name, _, qs = sys.argv[1].partition(":")
depths = sys.argv[2:] or ["0", "4"]
spec, q = config(name)
q = int(qs) if qs else q
inst = build_instance(spec)
c = inst.cds
w = torch.randn(q, c.n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
ref = None
s = torch.cuda.Stream()
for rep in range(2):
    for d0 in depths:
        os.environ["HMXG_PIPE"] = d0
        ev = Evaluator(c)  # the item list is built per evaluator and column count
        y = torch.full_like(w, float("nan"))
        for _ in range(3):
            ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(s)
        for _ in range(reps):
            ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=True, graph=False)
        torch.cuda.synchronize()
        dag = [p["ms"] for p in ev.phases() if p["kind"] == "dag"]
        if ref is None:
            ref = y.clone()
        same = bool(torch.equal(y, ref))
        print(f"{name} q={q} HMXG_PIPE={d0}: step {ms:.3f} ms, eval_dag {dag[0] if dag else float('nan'):.3f} ms, "
              f"same bits as the first: {same}", flush=True)
        ev.close()
