"""Regenerate the golden vectors from the REFERENCE library (oracle/_ref/libhmx_ref.so,
built from /root/reference/proj/src by oracle/Makefile). Run in the build container:

    python tests/golden/make_golden.py

Each case is a reference-built instance (tst::make_instance, proj/tests/helpers.hpp:101-118):
  cds/<name>.npz   the reference's own CDS (hmx::CDS arrays)
  <name>.npz       w, y_ref = hmx::evaluate(cds, plan{p=1}, w), y_evalref =
                   hmx::evaluate_reference(cm, w), y_dense = hmx::dense_apply(...)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402

CASES = {
    # acceptance criterion 1 (proj/tests/acceptance.cpp:74-91): exact HSS, eps_f 3.01e-14
    "crit1_hss_exact": (dict(n=512, d=2, kernel=0, h=5.0, sample_exact=1, bacc=0.0, leaf=64, max_rank=64, mode=1),
                        8, 1),
    # test_executor.cpp:190-212 shape (HSS, d=2, leaf 16)
    "hss_d2_n400": (dict(n=400, leaf=16, max_rank=24), 9, 2),
    # test_executor.cpp:167-188 shape (tau 0.65, d=8)
    "tau_d8_n420": (dict(n=420, d=8, leaf=16, max_rank=24, mode=0, tau=0.65, seed=3), 5, 3),
    # acceptance criterion 3 shape (d=32, tau, budget 64, knn 8, bacc 1e-3)
    "tau_d32_n400": (dict(n=400, d=32, leaf=64, max_rank=32, budget=64, knn_k=8, bacc=1e-3, mode=0, tau=0.65,
                           seed=105), 3, 105),
}


def main():
    os.makedirs(os.path.join(HERE, "cds"), exist_ok=True)
    for name, (kw, q, wseed) in CASES.items():
        ri = oracle.RefInstance(oracle.RefInstanceSpec(**kw))
        w = oracle.random_matrix(ri.cds.n, q, wseed)
        y_ref = ri.evaluate(w)
        y_er = ri.evaluate_reference(w)
        y_dense = ri.dense_apply(w)
        ri.cds.copy().save_npz(os.path.join(HERE, "cds", name + ".npz"))
        np.savez_compressed(os.path.join(HERE, name + ".npz"), w=w, y_ref=y_ref, y_evalref=y_er, y_dense=y_dense,
                            spec=np.array(repr(kw)))
        print(name, ri.cds.n, q, "evalref", oracle.rel_frob(y_er, y_ref), "dense", oracle.rel_frob(y_ref, y_dense))


if __name__ == "__main__":
    main()
