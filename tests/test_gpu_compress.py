"""GPU compression against the reference's own compress on the same
tree, samples, points and tolerance: identical ranks and skeletons everywhere, and bases
bit-identical for the inverse-distance kernel (correctly rounded operations only) or within
exp() rounding for the Gaussian (compress.cpp:17-148)."""
import numpy as np
import pytest

import oracle
from paper_1812_07152_b200.accuracy import Kernel
from paper_1812_07152_b200.compress import gpu_compress

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")]


def _gauss(x, y, h):
    d2 = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    return np.exp(-d2 / (2.0 * h * h))


def _compare(ri, kernel, exact):
    sp, si = ri.samples()
    pts = ri.points()
    bases = gpu_compress(pts, kernel, ri.cds, sp, si, ri.spec.bacc, ri.spec.max_rank)
    c = ri.cds
    ranks = []
    ref = [ri.basis(node) for node in range(c.num_nodes)]
    skel_ref = [r[1] for r in ref]
    for node in range(c.num_nodes):
        sr, sk, v = ref[node]
        b = bases[node]
        ranks.append(b.srank)
        assert b.srank == sr, node
        assert np.array_equal(b.skeleton, sk), node
        if not sr:
            continue
        assert b.v.shape == v.shape
        if exact:
            assert np.array_equal(b.v, v), node
            continue
        # Gaussian: entries differ from the host's exp() by ulps, which an ill-conditioned
        # R11 (bacc down to 1e-14) amplifies in V itself; the interpolation it defines does
        # not move: ||A - A[:, skel] V^T|| agrees with the reference's to rounding
        if c.lchild[node] == 0xFFFFFFFF:
            cols = c.perm[c.start[node]:c.end[node]]
        else:
            cols = np.concatenate([skel_ref[int(c.lchild[node])], skel_ref[int(c.rchild[node])]])
        a = _gauss(pts[si[sp[node]:sp[node + 1]]], pts[cols], kernel.h)
        a_sk = _gauss(pts[si[sp[node]:sp[node + 1]]], pts[sk], kernel.h)
        na = np.linalg.norm(a)
        res_ref = np.linalg.norm(a - a_sk @ v.T) / na
        res_gpu = np.linalg.norm(a - a_sk @ b.v.T) / na
        assert res_gpu <= max(1.5 * res_ref, 1e-13) and res_gpu <= 10 * max(ri.spec.bacc, 1e-14), node
    assert sum(ranks) > 0
    return ranks


@pytest.mark.parametrize("n,d,mode,tau,leaf,rank,seed,bacc", [
    (2000, 3, 1, 0.0, 64, 32, 1, 1e-5), (3000, 3, 0, 0.65, 64, 48, 2, 1e-7), (1500, 8, 1, 0.0, 32, 24, 3, 1e-3),
])
def test_invdist_bases_bitwise(n, d, mode, tau, leaf, rank, seed, bacc):
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=n, d=d, mode=mode, tau=tau, leaf=leaf, max_rank=rank, seed=seed,
                                                   kernel=1, bacc=bacc))
    _compare(ri, Kernel.inverse_distance(), exact=True)


@pytest.mark.parametrize("n,d,mode,h,bacc", [(2048, 3, 1, 0.5, 1e-5), (3000, 2, 0, 1.0, 1e-9), (1024, 4, 1, 2.0, 1e-3)])
def test_gaussian_bases_match(n, d, mode, h, bacc):
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=n, d=d, mode=mode, tau=0.65, leaf=64, max_rank=64, seed=4,
                                                   kernel=0, h=h, bacc=bacc))
    _compare(ri, Kernel.gaussian(h), exact=False)


@pytest.mark.parametrize("kernel,exact", [(1, True), (0, False)])
def test_gpu_inspector_p2_end_to_end(kernel, exact):
    """Tree, interactions and samples from the host; compression, every kernel block and
    the evaluation on the B200: the result is the reference's own CDS evaluated."""
    from paper_1812_07152_b200 import Evaluator
    from paper_1812_07152_b200.compress import cds_from_bases, skeleton_csr

    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=3000, d=3, mode=0, tau=0.65, leaf=64, max_rank=48, seed=9,
                                                   kernel=kernel, h=0.7, bacc=1e-6))
    k = Kernel.inverse_distance() if kernel else Kernel.gaussian(0.7)
    sp, si = ri.samples()
    bases = gpu_compress(ri.points(), k, ri.cds, sp, si, 1e-6, 48)
    cds = cds_from_bases(ri.cds, bases)
    if exact:
        assert np.array_equal(cds.vgen, ri.cds.vgen)
    ev = Evaluator(cds, points=ri.points(), kernel=k, skeletons=skeleton_csr(bases))
    w = oracle.random_matrix(3000, 16, 2)
    y = ev.evaluate(w)
    y_stored = Evaluator(ri.cds).evaluate(w)
    if exact:
        assert np.array_equal(y, y_stored)
    assert oracle.rel_frob(y, ri.evaluate(w)) <= 1e-12
