"""A/B of the eval_dag launch on one box (dev tool): device time of the DAG launch (per-launch
events, graph replay) for each library given, interleaved, in fresh processes.

    python tools/ab_dag.py cfg5-hss paper_1812_07152_b200/libhmxg.so build_ab/libhmxg_r1.so ...
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config
name = sys.argv[1]
spec, q = config(name)
inst = build_instance(spec)
ev = Evaluator(inst.cds)
w = torch.randn(q, inst.cds.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(w)
s = torch.cuda.Stream()
out = []
for k in range(13):
    ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=True, sync=True)
    if k >= 3:
        out.append([p["ms"] for p in ev.phases()])
print(json.dumps(out))
'''


def main():
    name, libs = sys.argv[1], sys.argv[2:]
    res = {lib: [] for lib in libs}
    for rep in range(2):
        for lib in libs:
            env = dict(os.environ, HMXG_LIBRARY=os.path.abspath(lib), ROOT=ROOT)
            r = subprocess.run([sys.executable, "-c", CHILD, name], capture_output=True, text=True, env=env)
            if r.returncode:
                print(lib, "failed", r.stderr[-500:])
                continue
            res[lib] += json.loads(r.stdout.strip().splitlines()[-1])
    for lib, rows in res.items():
        if not rows:
            continue
        cols = list(zip(*rows))
        print(f"{name} {os.path.basename(lib):24s} " + "  ".join(f"{min(c):.4f}/{sorted(c)[len(c)//2]:.4f}" for c in cols))


if __name__ == "__main__":
    main()
