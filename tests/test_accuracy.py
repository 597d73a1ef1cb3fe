"""The GPU error oracle: exact kernel products K(x_rows, :) W and the
relative error relative_error_vs, against the reference's own dense_apply /
relative_error_vs (executor.cpp:405-476) run on the same points, kernels and W."""
import numpy as np
import pytest

import oracle
from paper_1812_07152_b200 import InstanceSpec, build_instance
from paper_1812_07152_b200.accuracy import (DevicePoints, ErrorMode, Kernel, NumericGuardError, parse_kernel,
                                            relative_error, relative_error_vs, sample_rows)

needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


# ---------------------------------------------------------------- CPU
@needs_ref
@pytest.mark.parametrize("n,seed", [(1, 0), (100, 3), (256, 0), (257, 9), (4096, 42), (262144, 2**63 + 1)])
def test_sample_rows_match_reference(n, seed):
    assert np.array_equal(sample_rows(n, seed), oracle.ref_sample_rows(n, seed))


def test_parse_kernel():
    assert parse_kernel("gaussian:0.5") == Kernel("gaussian", 0.5)
    assert parse_kernel("invdist") == Kernel("invdist", 1.0)
    assert parse_kernel("exponential:2") == Kernel("exponential", 2.0)
    for bad in ("gaussian:0", "gaussian:-1", "cauchy:1"):
        with pytest.raises(ValueError):
            parse_kernel(bad)


# ---------------------------------------------------------------- GPU
def rel(a, b):
    return oracle.rel_frob(a, b)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("kernel,h,n,d,q", [(0, 1.0, 512, 2, 8), (0, 0.3, 2000, 3, 67), (1, 1.0, 1500, 4, 5),
                                            (0, 2.0, 777, 8, 130)])
def test_dense_apply_matches_reference(kernel, h, n, d, q):
    rng = np.random.default_rng(n)
    pts = rng.random((n, d))
    w = np.asfortranarray(rng.standard_normal((n, q)))
    y_ref = oracle.ref_dense_apply(pts, kernel, h, w)
    with DevicePoints(pts, Kernel("invdist" if kernel else "gaussian", h)) as dp:
        y = dp.dense_apply(w)
        assert rel(y, y_ref) <= 1e-13
        rows = rng.choice(n, size=77, replace=True).astype(np.uint32)
        assert rel(dp.kernel_rows(rows, w), y_ref[rows]) <= 1e-13
        # repeatable bit for bit (fixed split order, no atomics)
        assert np.array_equal(dp.dense_apply(w), y)


@pytest.mark.gpu
@needs_ref
def test_dense_apply_multiple_row_blocks():
    # n = 20000: the generated kernel tiles exceed one 2 GiB row block
    rng = np.random.default_rng(5)
    pts = rng.random((20000, 3))
    w = np.asfortranarray(rng.standard_normal((20000, 3)))
    y_ref = oracle.ref_dense_apply(pts, 0, 0.2, w)
    with DevicePoints(pts, Kernel.gaussian(0.2)) as dp:
        assert rel(dp.dense_apply(w), y_ref) <= 1e-13


@pytest.mark.gpu
def test_kernel_rows_exponential_matches_builder():
    inst = build_instance(InstanceSpec(n=6000, d=5, kernel="exponential", h=2.0, leaf=64, max_rank=32, seed=4))
    rng = np.random.default_rng(1)
    w = np.asfortranarray(rng.standard_normal((6000, 40)))
    rows = rng.choice(6000, size=300, replace=False).astype(np.uint32)
    with DevicePoints(inst.points(), Kernel.exponential(2.0)) as dp:
        assert rel(dp.kernel_rows(rows, w), inst.dense_rows(rows, w)) <= 1e-13
    inst.close()


@pytest.mark.gpu
def test_kernel_rows_device_pointers_equal_host():
    import torch

    rng = np.random.default_rng(2)
    pts = rng.random((3000, 3))
    w = np.asfortranarray(rng.standard_normal((3000, 70)))
    rows = rng.choice(3000, size=256, replace=False).astype(np.uint32)
    with DevicePoints(pts, Kernel.gaussian(0.4)) as dp:
        y_host = dp.kernel_rows(rows, w)
        wd = torch.from_numpy(w.T.copy()).cuda()       # n x q column major = (q, n) row major
        yd = torch.empty((70, 256), dtype=torch.float64, device="cuda")
        dp.kernel_rows_device(rows, wd.data_ptr(), yd.data_ptr(), 70)
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy().T, y_host)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("bacc,mode", [(1e-2, 0), (1e-3, 0), (1e-5, 0), (1e-3, 1), (1e-5, 1)])
def test_relative_error_matches_reference(bacc, mode):
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=2048, d=3, leaf=64, max_rank=64, bacc=bacc, seed=6, h=0.5))
    w = oracle.random_matrix(2048, 8, 3)
    y = ri.evaluate(w)
    eps_ref = ri.relative_error_vs(y, w, mode, seed=11)
    eps = relative_error_vs(y, Kernel.gaussian(0.5), ri.points(), w, ErrorMode(mode), seed=11)
    assert eps_ref > 1e-12
    assert abs(eps - eps_ref) <= 1e-6 * eps_ref
    # through the B200 evaluation (executor.cpp:478-483)
    eps2 = relative_error(ri.cds, Kernel.gaussian(0.5), ri.points(), w, ErrorMode(mode), seed=11)
    assert abs(eps2 - eps_ref) <= 1e-6 * eps_ref


@pytest.mark.gpu
@needs_ref
def test_relative_error_crit1_exact_instance():
    # proj/test_output.txt:21 — eps_f = 3.01e-14 for the exact HSS instance: at that level the
    # error is rounding noise, so the GPU's summation order may move it in the 2nd digit
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=512, d=2, kernel=0, h=5.0, sample_exact=1, bacc=0.0, leaf=64,
                                                   max_rank=64, mode=1))
    w = oracle.random_matrix(512, 8, 1)
    eps = relative_error(ri.cds, Kernel.gaussian(5.0), ri.points(), w, ErrorMode.DENSE)
    assert 1e-14 < eps < 1e-13


@pytest.mark.gpu
def test_relative_error_guard_and_empty():
    rng = np.random.default_rng(0)
    pts = rng.random((16385, 2))
    w = np.zeros((16385, 1))
    with pytest.raises(NumericGuardError):
        relative_error_vs(w, Kernel.gaussian(1.0), pts, w, ErrorMode.DENSE)
    with DevicePoints(pts, Kernel.gaussian(1.0)) as dp:
        with pytest.raises(NumericGuardError):
            dp.relative_error_vs(w, w, ErrorMode.DENSE)
        assert dp.relative_error_vs(np.zeros((16385, 0)), np.zeros((16385, 0)), ErrorMode.SAMPLED) == 0.0
        with pytest.raises(ValueError):
            dp.kernel_rows(None, np.zeros((10, 2)))


@pytest.mark.gpu
def test_sampled_error_full_size_cfg5():
    # BASELINE cfg5-HSS (n = 262144): 256 sampled exact rows against the builder's host rows
    from paper_1812_07152_b200 import config
    from paper_1812_07152_b200.executor import Evaluator

    spec, _ = config("cfg5-hss")
    inst = build_instance(spec)
    rng = np.random.default_rng(3)
    w = np.asfortranarray(rng.standard_normal((inst.cds.n, 16)))
    ev = Evaluator(inst.cds)
    y = ev.evaluate(w)
    with DevicePoints(inst.points(), Kernel.gaussian(spec.h)) as dp:
        rows = sample_rows(inst.cds.n, 7)
        exact = dp.kernel_rows(rows, w)
        assert rel(exact, inst.dense_rows(rows, w)) <= 1e-13
        eps = dp.relative_error_vs(y, w, ErrorMode.SAMPLED, seed=7)
        assert abs(eps - rel(y[rows], exact)) <= 1e-9 * eps
        # ranks saturate at s = 128 on depths 1-6, so the HSS approximation
        # of this h = 0.1 Gaussian is coarse: eps_f ~ 0.1 on the sampled rows
        assert 0.0 < eps < 0.5
    ev.close()
    inst.close()
