import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1812_07152_b200 import Evaluator, InstanceSpec, build_instance, config
inst = build_instance(InstanceSpec(n=3000, d=3, leaf=64, max_rank=48, mode="budget", budget=0.1, seed=4))
ev = Evaluator(inst.cds)
for q in [1, 2, 7, 8, 16, 33, 64, 65, 100, 128, 200]:
    w = np.asfortranarray(np.random.default_rng(q).standard_normal((inst.cds.n, q)))
    y = ev.evaluate(w)
    yr = oracle.oracle_evaluate(inst.cds, w)
    colerr = np.linalg.norm(y - yr, axis=0) / np.linalg.norm(yr, axis=0)
    print(q, oracle.rel_frob(y, yr), np.round(colerr[:10], 3))
