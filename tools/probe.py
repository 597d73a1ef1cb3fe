"""Device-resident timing of the evaluator on BASELINE configs with a per-launch breakdown (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

PEAK = 37.0e12
for name in sys.argv[1:] or ["cfg1-hss", "cfg5-hss"]:
    t = time.time()
    spec, q = config(name)
    inst = build_instance(spec)
    c = inst.cds
    ev = Evaluator(c)
    print(f"{name}: build {time.time()-t:.1f}s n={c.n} near={c.num_near} far={c.num_far} |D|={c.d_elems} |B|={c.b_elems} "
          f"|V|={c.v_elems} tiles={ev.info().device_bytes/1e9:.2f}GB", flush=True)
    w = torch.randn(q, c.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    s = torch.cuda.Stream()
    for _ in range(3):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    torch.cuda.synchronize()
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    e0.record(s)
    for _ in range(reps):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, levels=True)
    e1.record(s); torch.cuda.synchronize()
    ms_lv = e0.elapsed_time(e1) / reps
    ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=True, levels=True, graph=False)
    torch.cuda.synchronize()
    fl, by = c.flops(q), c.bytes(q)
    print(f"{name}: q={q} DAG {ms:.3f} ms {fl/ms/1e9:.2f} TFLOP/s eval-roofline frac={max(fl/PEAK, by/6555.8e9)*1e3/ms:.3f}"
          f" | level launches {ms_lv:.3f} ms")
    for p in ev.phases():
        f = p["flops_per_col"] * q
        print(f"   {p['kind']:>13} L{p['level']:<2} tiles={p['tiles']:>6} {p['ms']:.4f} ms {f/max(p['ms'],1e-9)/1e9:7.2f} TF/s")
    ev.close(); inst.close()
