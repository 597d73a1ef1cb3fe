"""CPU checks of the host side: the C-ABI libraries load and export every symbol the
headers declare, the CDS validation rejects malformed views with the reference's error
behaviour, and the instance builder produces CDSs with the reference's invariants."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from paper_1812_07152_b200 import (CDS, EvalPlan, EvalStats, InstanceSpec, PlanDefaults, build_instance, evaluate,
                                   generate_plan, plan_pseudocode)
from paper_1812_07152_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(hmx[gb]_\w+)\s*\(", text, re.M)))


@pytest.mark.parametrize("header,loader", [("hmxg.h", N.hmxg), ("hmxb.h", N.hmxb)])
def test_library_exports_every_declared_symbol(header, loader):
    lib = loader()
    names = _declared(header)
    assert len(names) >= 8
    for name in names:
        assert hasattr(lib, name), name
    table = N.HMXG_SYMBOLS if header == "hmxg.h" else N.HMXB_SYMBOLS
    assert set(names) == set(table)  # ctypes signatures cover the whole header


def _validate(cds: CDS):
    inf = N.Info()
    v = cds.view()
    rc = N.hmxg().hmxg_validate(C.byref(v), C.byref(inf))
    return rc, N.last_error(N.hmxg(), "hmxg"), inf


def _small():
    return build_instance(InstanceSpec(n=1500, d=3, leaf=40, max_rank=24, mode="budget", budget=0.1, h=0.4, seed=2))


def test_validate_accepts_builder_and_reference_cds():
    inst = _small()
    rc, _, inf = _validate(inst.cds)
    assert rc == 0
    assert inf.d_elems == inst.cds.d_elems and inf.b_elems == inst.cds.b_elems and inf.v_elems == inst.cds.v_elems
    assert inf.flops_per_col == pytest.approx(inst.cds.flops(1))
    if oracle.have_ref():
        ri = oracle.RefInstance(oracle.RefInstanceSpec(n=600, d=8, mode=0, tau=0.65, leaf=32, max_rank=24))
        assert _validate(ri.cds)[0] == 0


@pytest.mark.parametrize("breakage,needle", [
    ("perm", "bijection"), ("dptr", "near generator"), ("bptr", "far generator"), ("vptr", "V generator"),
    ("near_internal", "leaf pair"), ("child", "partition"), ("v_order", "no basis"),
])
def test_validate_rejects_malformed_views(breakage, needle):
    c = _small().cds.copy()
    if breakage == "perm":
        c.perm[0] = c.perm[1]
    elif breakage == "dptr":
        c.dptr[1] += 1
    elif breakage == "bptr":
        c.bptr[-1] += 1
    elif breakage == "vptr":
        c.vptr[1] += 1
    elif breakage == "near_internal":
        c.near_pairs[0, 1] = 1
    elif breakage == "child":
        c.end[int(c.lchild[0])] -= 1
    elif breakage == "v_order":
        c.v_order = c.v_order[:-1].copy()
        c.vptr = c.vptr[:-1].copy()
    rc, msg, _ = _validate(c)
    assert rc == N.HMXG_EINVAL
    assert needle in msg


def test_python_api_argument_errors_without_gpu():
    inst = _small()
    with pytest.raises(ValueError):
        evaluate(inst.cds, EvalPlan(), np.zeros((inst.cds.n + 1, 2)))
    st = EvalStats()
    y0 = evaluate(inst.cds, EvalPlan(), np.zeros((inst.cds.n, 0)), st)  # executor.cpp:279-282
    assert y0.shape == (inst.cds.n, 0) and st.locked_pairs == 0


def test_generate_plan_thresholds():
    inst = _small()
    plan = generate_plan(inst.cds, PlanDefaults(p=4))
    assert plan.block_threshold == len(inst.cds.leaves())
    assert plan.block_lowering_near == (inst.cds.num_near > plan.block_threshold)
    assert plan.coarsen_lowering == (inst.cds.height + 1 > 4)
    assert "pass upward" in plan_pseudocode(plan) and "pass near" in plan_pseudocode(plan)


def _leaf_cover(c: CDS):
    """Every ordered leaf pair must be covered exactly once by a near pair or by a far
    pair (i, j) with the leaves under i x j (the H-matrix block partition)."""
    leaves = c.leaves()
    lidx = {int(x): k for k, x in enumerate(leaves)}
    under = {}
    for i in range(c.num_nodes - 1, -1, -1):
        under[i] = [lidx[i]] if c.is_leaf(i) else under[int(c.lchild[i])] + under[int(c.rchild[i])]
    cover = np.zeros((len(leaves), len(leaves)), dtype=np.int64)
    for i, j in c.near_pairs:
        cover[lidx[int(i)], lidx[int(j)]] += 1
    for i, j in c.far_pairs:
        cover[np.ix_(under[int(i)], under[int(j)])] += 1
    return cover


@pytest.mark.parametrize("mode", ["hss", "tau", "budget"])
def test_builder_block_partition_and_symmetry(mode):
    inst = build_instance(InstanceSpec(n=2500, d=4, leaf=50, max_rank=20, mode=mode, budget=0.08, tau=0.65,
                                       h=0.5, seed=5))
    c = inst.cds
    assert np.array_equal(np.sort(c.perm), np.arange(c.n))
    assert np.all(_leaf_cover(c) == 1)
    near = {(int(i), int(j)) for i, j in c.near_pairs}
    far = {(int(i), int(j)) for i, j in c.far_pairs}
    assert all((j, i) in near for i, j in near) and all((j, i) in far for i, j in far)
    assert all((int(l), int(l)) in near for l in c.leaves())
    assert 0 not in {i for i, _ in near | far}  # the root never participates (interaction.cpp:145-157)


def test_builder_budget_near_fraction():
    inst = build_instance(InstanceSpec(n=20000, d=8, points="mixture", leaf=100, max_rank=32, mode="budget",
                                       budget=0.03, h=1.0, seed=42))
    c = inst.cds
    L = len(c.leaves())
    per_leaf = c.num_near / L
    target = int(np.ceil(0.03 * L))
    assert target <= per_leaf <= 2 * target  # symmetrization can only add


def test_builder_storage_order_and_generators():
    inst = _small()
    c = inst.cds
    # blocking order (structure.cpp:29-61): row group, column group, i, j
    bs = 2
    keys = [((int(i) - 1) // bs, (int(j) - 1) // bs, int(i), int(j)) for i, j in c.near_pairs]
    assert keys == sorted(keys)
    pts = inst.points()
    i, j = (int(x) for x in c.near_pairs[3])
    d = c.extract_d(3)
    pi, pj = pts[c.perm[c.start[i]:c.end[i]]], pts[c.perm[c.start[j]:c.end[j]]]
    dist2 = ((pi[:, None, :] - pj[None, :, :]) ** 2).sum(-1)
    assert np.allclose(d, np.exp(-dist2 / (2 * 0.4 ** 2)), rtol=1e-14, atol=0)
    # nested basis: identity rows at the skeleton positions
    node = int(c.v_order[0])
    v = c.extract_v(node)
    assert v.shape == (c.v_width(node), int(c.sranks[node]))
    assert np.sum(np.isclose(v, 1.0).all(axis=1) | True) >= 0
    eye_rows = [r for r in range(v.shape[0]) if np.count_nonzero(v[r]) == 1 and np.isclose(v[r].max(), 1.0)]
    assert len(eye_rows) >= v.shape[1]


def test_builder_points_generators():
    from paper_1812_07152_b200.instance import InstanceSpec as S
    p = build_instance(S(n=5000, d=28, points="normal", leaf=256, max_rank=8, h=3.0, seed=1)).points()
    assert np.allclose(p.mean(0), 0.0, atol=1e-12) and np.allclose(p.std(0), 1.0, atol=1e-12)
    q = build_instance(S(n=3000, d=64, points="quantized", leaf=256, max_rank=8, kernel="exponential", h=2.0,
                         seed=1)).points()
    assert len(np.unique(q)) == 16 and q.min() == 0.0 and q.max() == 1.0
    if oracle.have_ref():  # uniform points equal the reference synth_points bit for bit
        ri = oracle.RefInstance(oracle.RefInstanceSpec(n=700, d=3, leaf=64, seed=42))
        ptr = C.POINTER(C.c_double)()
        n, d = C.c_uint64(), C.c_uint64()
        oracle._ref_lib().hmxr_points(ri._h, C.byref(ptr), C.byref(n), C.byref(d))
        ref_pts = np.ctypeslib.as_array(ptr, shape=(700, 3)).copy()
        mine = build_instance(S(n=700, d=3, leaf=64, max_rank=8, seed=42)).points()
        assert np.array_equal(ref_pts, mine)


def test_builder_rejects_bad_specs():
    with pytest.raises(ValueError):
        build_instance(InstanceSpec(n=100, leaf=100))  # one-node tree (structure.cpp:35-36)
    with pytest.raises(ValueError):
        build_instance(InstanceSpec(n=100, leaf=10, h=-1.0))


def test_builder_accuracy_tracks_tolerance():
    # the compression is a real approximation: eps_f shrinks with the tolerance
    # (acceptance criterion 2 analogue, proj/tests/acceptance.cpp:95-121)
    errs = []
    for tol in (1e-2, 1e-5):
        inst = build_instance(InstanceSpec(n=2048, d=2, leaf=128, max_rank=128, mode="hss", h=1.0, tol=tol,
                                           sample_rows=256, seed=1))
        w = np.asfortranarray(np.random.default_rng(2).standard_normal((2048, 4)))
        y = oracle.oracle_evaluate(inst.cds, w)
        rows = np.arange(0, 2048, 4, dtype=np.uint32)
        exact = inst.dense_rows(rows, w)
        errs.append(np.linalg.norm(y[rows] - exact) / np.linalg.norm(exact))
    assert errs[1] < errs[0] and errs[1] < 1e-3


def test_identity_rows_lowering_counts():
    """The plan drops exactly the multiply-adds of the bases' unit rows (plan.cpp
    identity rows): executed flops = reference flops - 2 x 2 x (unit-row elements of every
    active node's V), once upward and once downward."""
    import ctypes as C

    import numpy as np

    from paper_1812_07152_b200 import InstanceSpec, build_instance
    from paper_1812_07152_b200 import _native as N

    inst = build_instance(InstanceSpec(n=6000, d=3, leaf=64, max_rank=48, seed=8))
    c = inst.cds
    unit = 0
    for node in range(c.num_nodes):
        if c.sranks[node] == 0 or not c.participating[node]:
            continue
        v = c.extract_v(node)
        claimed = set()
        for r in v:  # a unit row claims its column once (plan.cpp)
            nz = np.flatnonzero(r)
            if nz.size == 1 and r[nz[0]] == 1.0 and nz[0] not in claimed:
                claimed.add(nz[0])
                unit += v.shape[1]
    info = N.Info()
    view = c.view()
    assert N.hmxg().hmxg_validate(C.byref(view), C.byref(info)) == N.HMXG_OK
    assert unit > 0
    assert info.exec_flops_per_col == pytest.approx(info.flops_per_col - 2 * 2 * unit, rel=1e-12)
    inst.close()


@pytest.mark.parametrize("q,grid", [(1, 444), (64, 444), (65, 444), (256, 444), (2048, 444), (256, 4), (256, 100000)])
def test_dag_claim_order_is_topological(q, grid):
    """eval_dag's deadlock freedom (DESIGN, Kernels): in the claim order every tile an item
    waits for comes first, each task tile of the leaf variant that runs appears once, and
    the completion targets equal the writer tile counts. Host-only (hmxg_dag_check); the
    grid sizes pick the combined (few CTAs) or split (many CTAs) leaf variant."""
    insts = [_small(),
             build_instance(InstanceSpec(n=3000, d=3, leaf=48, max_rank=40, mode="tau", tau=0.7, seed=12)),
             build_instance(InstanceSpec(n=2000, d=2, leaf=32, max_rank=16, seed=5))]
    for inst in insts:
        v = inst.cds.view()
        n_items = C.c_uint64()
        rc = N.hmxg().hmxg_dag_check(C.byref(v), q, grid, C.byref(n_items))
        assert rc == 0, N.last_error(N.hmxg(), "hmxg")
        assert n_items.value > 0
        inst.close()


def test_dag_claim_order_reference_instance():
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=460, d=8, mode=0, tau=0.65, leaf=16, max_rank=24, seed=4))
    v = ri.cds.view()
    for q, grid in [(7, 444), (130, 444), (130, 2)]:
        assert N.hmxg().hmxg_dag_check(C.byref(v), q, grid, None) == 0, N.last_error(N.hmxg(), "hmxg")


@pytest.mark.parametrize("name", ["cfg1-hss", "cfg2-h2b", "cfg5-hss"])
def test_dag_claim_order_baseline_configs(name):
    """(cfg5-hss at Q=2048 is the headline: 663 work items per CTA, the subtree-pipelined order.)"""
    from paper_1812_07152_b200 import config

    spec, q = config(name)
    inst = build_instance(spec)
    v = inst.cds.view()
    for qq in (q,) if name == "cfg5-hss" else (q, 4 * q):
        assert N.hmxg().hmxg_dag_check(C.byref(v), qq, 444, None) == 0, N.last_error(N.hmxg(), "hmxg")
    inst.close()


def test_cds_fingerprint_sees_every_edit():
    """hmxg_cds_fingerprint (the drop-in caches' key): stable across calls and copies, and
    changed by a one-ulp edit of any generator, a structure edit, or a different CDS."""
    inst = _small()
    cds = inst.cds
    fp = cds.fingerprint()
    assert fp == cds.fingerprint()
    for name in ("dgen", "bgen", "vgen"):
        arr = getattr(cds, name)
        k = arr.size // 2
        old = arr[k]
        arr[k] = np.nextafter(old, np.inf)
        assert cds.fingerprint() != fp, name
        arr[k] = old
        assert cds.fingerprint() == fp
    cds.perm[[0, 1]] = cds.perm[[1, 0]]
    assert cds.fingerprint() != fp
    cds.perm[[0, 1]] = cds.perm[[1, 0]]
    other = build_instance(InstanceSpec(n=1500, d=3, leaf=40, max_rank=24, mode="budget", budget=0.1, h=0.4, seed=3))
    assert other.cds.fingerprint() != fp


def test_dag_check_ctree_mode(monkeypatch):
    """CTree mode (HMXG_CTREE=1): the item list is the near tiles only (x column blocks x
    parts), and the CTree levels hold every other task of the split variant once, each level
    reading only rows of earlier levels (hmxg_dag_check's CTree branch). (CTree runs the
    level-by-level tree: the flat tree of small trees is off.)"""
    from paper_1812_07152_b200 import config

    monkeypatch.setenv("HMXG_NO_FLAT", "1")

    insts = [build_instance(config("cfg1-hss")[0]), _small(),
             build_instance(InstanceSpec(n=1500, d=5, leaf=40, max_rank=24, mode="budget", budget=0.1, seed=9))]
    for inst in insts:
        v = inst.cds.view()
        for q in (8, 37, 64, 100):
            n_dag, n_ct = C.c_uint64(), C.c_uint64()
            monkeypatch.delenv("HMXG_CTREE", raising=False)
            assert N.hmxg().hmxg_dag_check(C.byref(v), q, 444, C.byref(n_dag)) == 0, N.last_error(N.hmxg(), "hmxg")
            monkeypatch.setenv("HMXG_CTREE", "1")
            assert N.hmxg().hmxg_dag_check(C.byref(v), q, 444, C.byref(n_ct)) == 0, N.last_error(N.hmxg(), "hmxg")
            assert 0 < n_ct.value < n_dag.value  # the near tiles only
        inst.close()


@pytest.mark.parametrize("frac", ["0.1", "0.35", "1"])
def test_dag_check_partial_split(frac, monkeypatch):
    """A partial split (HMXG_SPLIT_FRAC): a fraction of the leaves run as split-variant near
    tiles between the tree levels plus accumulating tiles at the end, the rest as combined
    tiles; the claim order stays topological and every tile appears once per column block."""
    from paper_1812_07152_b200 import config

    monkeypatch.setenv("HMXG_SPLIT_FRAC", frac)
    insts = [build_instance(config("cfg1-hss")[0]), _small(),
             build_instance(InstanceSpec(n=3000, d=3, leaf=48, max_rank=40, mode="budget", budget=0.1, seed=12))]
    for inst in insts:
        v = inst.cds.view()
        for q, grid in [(2048, 444), (640, 444), (64, 2)]:
            assert N.hmxg().hmxg_dag_check(C.byref(v), q, grid, None) == 0, N.last_error(N.hmxg(), "hmxg")
        inst.close()


@pytest.mark.parametrize("d0", ["1", "2", "3"])
def test_dag_check_subtree_pipelined_order(d0, monkeypatch):
    """The subtree-pipelined claim order of wide DAGs (HMXG_PIPE = the grouping depth d0): the
    far+downward levels of one group of subtrees interleaved with the previous group's leaf
    rows. Still every tile once per
    column block and topological, on balanced, uneven (two-means) and cross-level (tau, budget)
    trees; the item count equals the level-major order's."""
    monkeypatch.setenv("HMXG_NO_FLAT", "1")
    monkeypatch.setenv("HMXG_PIPE_MIN", "1")
    insts = [build_instance(InstanceSpec(n=4096, d=3, leaf=32, max_rank=24, seed=2)),
             build_instance(InstanceSpec(n=5000, d=2, leaf=40, max_rank=30, seed=3, split="twomeans")),
             build_instance(InstanceSpec(n=6000, d=3, leaf=48, max_rank=40, mode="budget", budget=0.1, seed=12)),
             build_instance(InstanceSpec(n=5000, d=3, leaf=48, max_rank=40, mode="tau", tau=0.6, seed=7))]
    for inst in insts:
        v = inst.cds.view()
        for q, grid in [(2048, 444), (200, 4), (64, 1)]:
            n_pipe, n_level = C.c_uint64(), C.c_uint64()
            monkeypatch.setenv("HMXG_PIPE", d0)
            assert N.hmxg().hmxg_dag_check(C.byref(v), q, grid, C.byref(n_pipe)) == 0, N.last_error(N.hmxg(), "hmxg")
            monkeypatch.setenv("HMXG_PIPE", "0")
            assert N.hmxg().hmxg_dag_check(C.byref(v), q, grid, C.byref(n_level)) == 0, N.last_error(N.hmxg(), "hmxg")
            assert n_pipe.value == n_level.value > 0
        # the two orders are permutations of one another
        n = n_level.value
        a, b = (C.c_uint64 * n)(), (C.c_uint64 * n)()
        monkeypatch.setenv("HMXG_PIPE", d0)
        assert N.hmxg().hmxg_dag_items(C.byref(v), 64, 1, a, n, None) == 0
        monkeypatch.setenv("HMXG_PIPE", "0")
        assert N.hmxg().hmxg_dag_items(C.byref(v), 64, 1, b, n, None) == 0
        assert list(a) != list(b) and sorted(a) == sorted(b)
        inst.close()
