"""Generated near field (include/hmxg.h hmxg_upload_generated): the near
blocks D_ij are evaluated on the device from the points instead of shipped from the host.

* inverse distance uses only correctly rounded operations, so the generated D equals the
  host-built D bit for bit and so does Y;
* Gaussian / exponential differ from the host's exp() by at most an ulp per entry;
* a reference-built CDS evaluated with its D generated on the GPU matches the reference's
  own hmx::evaluate to the north-star tolerance."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1812_07152_b200 import Evaluator, InstanceSpec, build_instance
from paper_1812_07152_b200 import _native as N
from paper_1812_07152_b200.accuracy import Kernel

TOL = 1e-12


def _pair(kernel, h, **kw):
    spec = InstanceSpec(n=4000, d=3, kernel=kernel, h=h, leaf=64, max_rank=32, seed=5, **kw)
    full = build_instance(spec)
    spec.skip_near = True
    lean = build_instance(spec)
    assert lean.cds.dgen.size == 0 and full.cds.dgen.size == int(full.cds.dptr[-1]) > 0
    assert np.array_equal(lean.cds.dptr, full.cds.dptr)
    return full, lean


def test_plain_upload_refuses_missing_near_field():
    _, lean = _pair("gaussian", 0.5)
    v = lean.cds.view()
    assert N.hmxg().hmxg_validate(C.byref(v), None) == N.HMXG_EINVAL


@pytest.mark.gpu
def test_invdist_generated_is_bitwise_equal():
    full, lean = _pair("invdist", 1.0, mode="tau", tau=0.65)
    w = np.asfortranarray(np.random.default_rng(1).standard_normal((4000, 37)))
    y_stored = Evaluator(full.cds).evaluate(w)
    y_gen = Evaluator(lean.cds, points=lean.points(), kernel=Kernel.inverse_distance()).evaluate(w)
    assert np.array_equal(y_gen, y_stored)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,h,mode", [("gaussian", 0.5, "hss"), ("exponential", 2.0, "budget"),
                                           ("gaussian", 0.3, "budget")])
def test_generated_matches_stored(kernel, h, mode):
    full, lean = _pair(kernel, h, mode=mode)
    w = np.asfortranarray(np.random.default_rng(2).standard_normal((4000, 70)))
    y_stored = Evaluator(full.cds).evaluate(w)
    ev = Evaluator(lean.cds, points=lean.points(), kernel=Kernel(kernel, h))
    y_gen = ev.evaluate(w)
    assert oracle.rel_frob(y_gen, y_stored) <= 1e-14
    assert oracle.rel_frob(y_gen, oracle.oracle_evaluate(full.cds, w)) <= TOL
    # the lean device copy holds the same pre-tiled operands; the host never held D
    assert ev.info().d_elems == int(full.cds.dptr[-1])


@pytest.mark.gpu
def test_reference_cds_with_generated_near_field():
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=3000, d=3, mode=0, tau=0.65, leaf=64, max_rank=48, seed=9, h=0.7))
    w = oracle.random_matrix(3000, 24, 4)
    ev = Evaluator(ri.cds, points=ri.points(), kernel=Kernel.gaussian(0.7))
    assert oracle.rel_frob(ev.evaluate(w), ri.evaluate(w)) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,h,mode,scratch_mb", [("gaussian", 0.5, "hss", "1"), ("exponential", 2.0, "budget", "2"),
                                                      ("invdist", 1.0, "tau", "4096")])
def test_near_on_the_fly_equals_resident(kernel, h, mode, scratch_mb, monkeypatch):
    """HMXG_UPLOAD_NEAR_ON_THE_FLY: the near blocks are never resident; every evaluation
    generates them wave by wave into the scratch (a 1-2 MB scratch forces many waves) right
    before the wave's leaf rows. Y is bit-identical to the resident generated near field on
    the DAG and level-launch sequences, host and device paths; the resident bytes drop by the
    near blocks, and the launch sequence reports one generation + one leaf launch per wave."""
    import torch

    from paper_1812_07152_b200.executor import torch_stream

    kw = {"tau": 0.65} if mode == "tau" else {}
    _, lean = _pair(kernel, h, mode=mode, **kw)
    kern = Kernel.inverse_distance() if kernel == "invdist" else Kernel(kernel, h)
    w = np.asfortranarray(np.random.default_rng(3).standard_normal((4000, 70)))
    res = Evaluator(lean.cds, points=lean.points(), kernel=kern)
    y_res = res.evaluate(w)
    monkeypatch.setenv("HMXG_NEAR_SCRATCH_MB", scratch_mb)
    otf = Evaluator(lean.cds, points=lean.points(), kernel=kern, near_on_the_fly=True)
    assert np.array_equal(otf.evaluate(w), y_res)
    assert np.array_equal(otf.evaluate(w, levels=True), y_res)
    wd = torch.from_numpy(w.T.copy()).cuda()
    yd = torch.full_like(wd, float("nan"))
    for graph in (False, True, True):
        otf.evaluate_device(wd.data_ptr(), yd.data_ptr(), 70, stream=torch_stream(), graph=graph, sync=True,
                            time_phases=True)
        assert np.array_equal(yd.cpu().numpy().T, y_res)
    kinds = [p["kind"] for p in otf.phases()]
    waves = kinds.count("near-gen")
    assert waves >= (2 if scratch_mb in ("1", "2") else 1) and kinds.count("near+leaf") == waves
    if waves > 1:  # the scratch holds one wave's near blocks, not all of them
        assert otf.info().device_bytes < res.info().device_bytes
    assert kinds[0] == "gather" and kinds[-1] == "scatter" and all(p["ms"] > 0 for p in otf.phases())
    assert oracle.rel_frob(y_res, oracle.oracle_evaluate(_pair(kernel, h, mode=mode, **kw)[0].cds, w)) <= TOL
    res.close()
    otf.close()


@pytest.mark.gpu
def test_near_on_the_fly_without_tree_levels():
    """A tau tree whose blocks are all near (every rank 0) has no DAG items once the near field
    runs in on-the-fly waves: the empty item list is a prepared list, not an error (found by
    tests/test_gpu_fuzz.py), and repeated calls reuse it."""
    spec = InstanceSpec(n=1184, d=5, kernel="exponential", h=0.5, leaf=33, mode="tau", tau=0.9, max_rank=24,
                        split="kd", seed=11)
    full = build_instance(spec)
    assert int(full.cds.sranks.max()) == 0 and full.cds.num_far == 0
    spec.skip_near = True
    lean = build_instance(spec)
    w = np.asfortranarray(np.random.default_rng(6).standard_normal((spec.n, 70)))
    otf = Evaluator(lean.cds, points=lean.points(), kernel=Kernel("exponential", 0.5), near_on_the_fly=True)
    y = otf.evaluate(w)
    assert np.array_equal(otf.evaluate(w), y)
    assert oracle.rel_frob(y, oracle.oracle_evaluate(full.cds, w)) <= TOL
    otf.close()
