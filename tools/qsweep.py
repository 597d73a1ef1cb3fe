"""Per-Q device timing of one config (dev tool): the per-GPU column shard of the scaling
run is Q/N, so this shows how the evaluation rate holds up as the shard narrows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5-hss"
qs = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2048, 1024, 512, 256, 128, 64]
spec, _ = config(name)
inst = build_instance(spec)
c = inst.cds
ev = Evaluator(c)
s = torch.cuda.Stream()
for q in qs:
    w = torch.randn(q, c.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    for _ in range(3):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    torch.cuda.synchronize()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=True, graph=False)
    torch.cuda.synchronize()
    ph = " ".join(f"{p['kind']}={p['ms']:.3f}" for p in ev.phases())
    print(f"{name} q={q}: {ms:.3f} ms {c.flops(q)/ms/1e9:.2f} TFLOP/s | {ph}", flush=True)
    del w, y
