"""One device-resident evaluation of a config (target for ncu captures)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5-hss")
ap.add_argument("--q", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--levels", action="store_true", help="the level-by-level launch sequence (grouped_gemm per level)")
a = ap.parse_args()
spec, q = config(a.config)
q = a.q or q
inst = build_instance(spec)
ev = Evaluator(inst.cds)
w = torch.randn((q, inst.cds.n), dtype=torch.float64, device="cuda")
y = torch.empty_like(w)
for _ in range(a.reps):
    ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, sync=True, levels=a.levels)
torch.cuda.synchronize()
print("launches per eval", ev.info().launches_per_eval, "grouped_gemm per eval", ev.info().launches_per_eval - 2)
