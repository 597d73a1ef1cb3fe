"""One device-resident evaluation with the near field on the fly (target of ncu captures of gen_near)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config
from paper_1812_07152_b200.accuracy import Kernel

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2-h2b"
spec, q = config(name)
spec.skip_near = True
inst = build_instance(spec)
ev = Evaluator(inst.cds, points=inst.points(), kernel=Kernel(spec.kernel, spec.h), near_on_the_fly=True)
w = torch.randn((q, inst.cds.n), dtype=torch.float64, device="cuda")
y = torch.empty_like(w)
ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, sync=True)
torch.cuda.synchronize()
print("ok", [p["kind"] for p in ev.phases()])
