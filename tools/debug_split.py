"""Split-mode evaluation vs the single-device one, repeated on fresh parts (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config
from paper_1812_07152_b200.distributed import SplitPart, split_evaluate
from paper_1812_07152_b200.executor import torch_stream
spec, _ = config(sys.argv[1] if len(sys.argv) > 1 else "cfg2-h2b"); inst = build_instance(spec); n = inst.cds.n
q = int(sys.argv[2]) if len(sys.argv) > 2 else 128
w = torch.randn((q, n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
ev = Evaluator(inst.cds); yf = torch.empty_like(w)
ev.evaluate_device(w.data_ptr(), yf.data_ptr(), q, sync=True, stream=torch_stream())
for nparts in (2, 3, 4):
    parts = [SplitPart(inst.cds, nparts, k) for k in range(nparts)]
    for rep in range(3):
        y = split_evaluate(inst.cds, w, parts=parts); torch.cuda.synchronize()
        d = (y - yf).abs(); bad = (d > 0).nonzero()
        print(nparts, rep, "maxdiff", float(d.max()), "bad", bad.shape[0], "rel", float(d.norm() / yf.norm()), flush=True)
    for p in parts:
        p.close()
