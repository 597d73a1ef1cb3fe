"""Quick device-resident timing of the evaluator on BASELINE configs (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

PEAK = 37.0e12
for name in sys.argv[1:] or ["cfg1-hss", "cfg5-hss"]:
    t = time.time()
    spec, q = config(name)
    inst = build_instance(spec)
    c = inst.cds
    print(f"{name}: build {time.time()-t:.1f}s n={c.n} nodes={c.num_nodes} near={c.num_near} far={c.num_far} "
          f"|D|={c.d_elems} |B|={c.b_elems} |V|={c.v_elems} maxsr={c.sranks.max()} {inst.stats['seconds_compress']:.1f}s compress", flush=True)
    ev = Evaluator(c)
    w = torch.randn(q, c.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    for _ in range(3):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record(s)
    for _ in range(reps):
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream)
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = c.flops(q); by = c.bytes(q)
    print(f"{name}: q={q} {ms:.3f} ms  {fl/ms/1e6:.1f} GFLOP/s  frac_fp64={fl/ms/1e9/PEAK*1e3*1e-3:.3f} "
          f"roofline_ms={max(fl/PEAK, by/6555.8e9)*1e3:.3f}", flush=True)
    ev.close(); inst.close()
