"""GPU parity of the B200 evaluator against the oracle (reference restatement, reference
library, committed golden vectors). Tolerance: relative Frobenius error <= 1e-12 (FP64,
BASELINE.json north_star); integer-exact properties (K = I, zero W, column independence,
run-to-run determinism) are checked bit for bit."""
import glob
import os

import numpy as np
import pytest

import oracle
from paper_1812_07152_b200.executor import torch_stream
from paper_1812_07152_b200 import CDS, EvalPlan, EvalStats, Evaluator, InstanceSpec, build_instance, config, evaluate

pytestmark = pytest.mark.gpu
TOL = 1e-12
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _w(n, q, seed):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((n, q)))


REF_SPECS = [
    # (n, d, mode, tau, leaf, max_rank, seed) — shapes of proj/tests/test_executor.cpp:30-130
    (512, 2, 1, 0.0, 64, 64, 1),
    (340, 2, 1, 0.0, 16, 24, 1),
    (380, 8, 0, 0.65, 16, 24, 2),
    (460, 8, 0, 0.65, 16, 24, 4),
    (2048, 32, 0, 0.65, 64, 32, 9),
    (4096, 3, 1, 0.0, 128, 64, 42),
]


@pytest.mark.parametrize("n,d,mode,tau,leaf,rank,seed", REF_SPECS)
def test_reference_instances(n, d, mode, tau, leaf, rank, seed):
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=n, d=d, mode=mode, tau=tau, leaf=leaf, max_rank=rank,
                                                   seed=seed))
    w = oracle.random_matrix(n, 7, seed)
    y_ref = ri.evaluate(w)
    stats = EvalStats()
    y = evaluate(ri.cds, EvalPlan(), w, stats)
    assert oracle.rel_frob(y, y_ref) <= TOL
    assert oracle.rel_frob(y, ri.evaluate_reference(w)) <= 1e-13 * 10
    assert stats.locked_pairs == 0 and stats.seconds >= 0.0 and stats.launches > 0


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))))
def test_golden_vectors(path):
    z = np.load(path)
    cds = CDS.load_npz(os.path.join(GOLDEN, "cds", os.path.basename(path)))
    y = evaluate(cds, EvalPlan(), z["w"])
    assert oracle.rel_frob(y, z["y_ref"]) <= TOL


@pytest.mark.parametrize("name", ["cfg1-hss", "cfg2-h2b"])
def test_configs_full(name):
    spec, q = config(name)
    inst = build_instance(spec)
    w = _w(inst.cds.n, q, 5)
    y = Evaluator(inst.cds).evaluate(w)
    assert oracle.rel_frob(y, oracle.oracle_evaluate(inst.cds, w)) <= TOL


def test_exponential_kernel_and_ragged_leaves():
    inst = build_instance(InstanceSpec(n=6000, d=16, points="quantized", kernel="exponential", h=2.0, leaf=100,
                                       mode="budget", budget=0.08, max_rank=48, tol=1e-5, seed=3))
    sizes = inst.cds.end - inst.cds.start
    leaves = inst.cds.leaves()
    assert len(set(sizes[leaves].tolist())) > 1  # two-means: ragged leaves
    w = _w(inst.cds.n, 37, 1)  # ragged Q as well
    y = Evaluator(inst.cds).evaluate(w)
    assert oracle.rel_frob(y, oracle.oracle_evaluate(inst.cds, w)) <= TOL


def test_identity_kernel_is_bitwise():
    # proj/tests/test_executor.cpp:117-130: an underflowing Gaussian on the integer grid
    inst = build_instance(InstanceSpec(n=100, points="grid2d", h=0.01, leaf=8, max_rank=16, seed=1))
    assert int(inst.cds.sranks.max()) == 0
    w = _w(100, 4, 5)
    assert np.array_equal(evaluate(inst.cds, EvalPlan(), w), w)


def test_zero_and_empty():
    inst = build_instance(InstanceSpec(n=200, d=2, leaf=32, max_rank=32, seed=1))
    y0 = evaluate(inst.cds, EvalPlan(), np.zeros((200, 0)))
    assert y0.shape == (200, 0)
    yz = evaluate(inst.cds, EvalPlan(), np.zeros((200, 3)))
    assert np.all(yz == 0.0)
    with pytest.raises(ValueError):
        evaluate(inst.cds, EvalPlan(), np.zeros((201, 2)))


def test_linearity():
    inst = build_instance(InstanceSpec(n=3500, d=3, leaf=64, max_rank=48, mode="budget", budget=0.1, seed=4))
    ev = Evaluator(inst.cds)
    w1, w2 = _w(3500, 3, 11), _w(3500, 3, 12)
    y1, y2, yc = ev.evaluate(w1), ev.evaluate(w2), ev.evaluate(2.75 * w1 + w2)
    assert oracle.rel_frob(yc, 2.75 * y1 + y2) <= TOL


def test_bitwise_determinism_and_column_independence():
    spec, _ = config("cfg1-hss")
    inst = build_instance(spec)
    ev = Evaluator(inst.cds)
    w = _w(inst.cds.n, 150, 2)
    a = ev.evaluate(w)
    assert np.array_equal(a, ev.evaluate(w))
    cols = [0, 3, 64, 65, 149]
    sub = ev.evaluate(np.asfortranarray(w[:, cols]))
    assert np.array_equal(sub, a[:, cols])  # Y[:,c] depends only on W[:,c]


def test_column_sharded_context_matches_single_device():
    # two column shards on the same physical GPU exercise the multi-device split path
    spec, _ = config("cfg1-hss")
    inst = build_instance(spec)
    w = _w(inst.cds.n, 130, 3)
    one = Evaluator(inst.cds, devices=(0,)).evaluate(w)
    two = Evaluator(inst.cds, devices=(0, 0)).evaluate(w)
    assert np.array_equal(one, two)


def test_device_pointer_path():
    import torch

    spec, _ = config("cfg1-hss")
    inst = build_instance(spec)
    w = _w(inst.cds.n, 64, 4)
    ev = Evaluator(inst.cds)
    wd = torch.from_numpy(w.T.copy()).cuda()  # (q, n) row major == n x q column major
    yd = torch.empty_like(wd)
    ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), 64, stream=torch_stream())
    torch.cuda.synchronize()
    y = yd.cpu().numpy().T
    assert np.array_equal(y, ev.evaluate(w))


@pytest.mark.parametrize("name,q", [("cfg5-hss", 320), ("cfg2-h2b", 1024)])
def test_leaf_variants_give_the_same_bits(name, q):
    """Wide Q on the device runs the combined leaf tasks (≥48 work items per CTA); the host
    path evaluates 64-column chunks, which run the split leaf variant (near tasks, then
    V_i S_i accumulated). Both sum every row in one order: equal bit for bit."""
    import torch

    spec, _ = config(name)
    inst = build_instance(spec)
    n = inst.cds.n
    ev = Evaluator(inst.cds)
    w = _w(n, q, 8)
    wd = torch.from_numpy(w.T.copy()).cuda()
    yd = torch.empty_like(wd)
    ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=torch_stream())
    torch.cuda.synchronize()
    y_dev = yd.cpu().numpy().T
    assert np.array_equal(y_dev, ev.evaluate(w))
    assert np.array_equal(y_dev, ev.evaluate(w, levels=True))
    cols = np.arange(0, q, q // 16)
    assert oracle.rel_frob(y_dev[:, cols], oracle.oracle_evaluate(inst.cds, np.asfortranarray(w[:, cols]))) <= TOL


def test_graph_replay_matches_direct_launches():
    import torch

    spec, _ = config("cfg2-h2b")
    inst = build_instance(spec)
    n, q = inst.cds.n, 96
    ev = Evaluator(inst.cds)
    s = torch.cuda.Stream()
    w = torch.randn((q, n), dtype=torch.float64, device="cuda")
    y_direct, y_graph = torch.empty_like(w), torch.empty_like(w)
    s.wait_stream(torch.cuda.current_stream())  # W is written on torch's stream
    ev.evaluate_device(w.data_ptr(), y_direct.data_ptr(), q, stream=s.cuda_stream, sync=True, graph=False)
    for _ in range(2):  # capture, then replay
        ev.evaluate_device(w.data_ptr(), y_graph.data_ptr(), q, stream=s.cuda_stream, sync=True)
    assert torch.equal(y_direct, y_graph)
    w.copy_(torch.randn_like(w))  # same pointers, new data: the replay must read it
    s.wait_stream(torch.cuda.current_stream())
    ev.evaluate_device(w.data_ptr(), y_graph.data_ptr(), q, stream=s.cuda_stream, sync=True)
    ev.evaluate_device(w.data_ptr(), y_direct.data_ptr(), q, stream=s.cuda_stream, sync=True, graph=False)
    assert torch.equal(y_direct, y_graph)
    y = y_graph.cpu().numpy().T
    assert oracle.rel_frob(y, oracle.oracle_evaluate(inst.cds, w.cpu().numpy().T)) <= TOL


def _ref_columns(cds, w, threads=None):
    """The reference library's hmx::evaluate (oracle/_ref, p = 1: no WorkerPool threads, so no
    F5 hang) on column chunks in parallel host threads; every column is computed by the same
    arithmetic whatever the chunk (the reference's GEMMs loop columns outermost)."""
    from concurrent.futures import ThreadPoolExecutor

    ref = oracle.RefCds(cds)
    q = w.shape[1]
    threads = threads or min(q, os.cpu_count() or 1)
    cuts = [q * k // threads for k in range(threads + 1)]
    out = np.empty_like(w)

    def run(k):
        a, b = cuts[k], cuts[k + 1]
        if b > a:
            out[:, a:b] = ref.evaluate(np.asfortranarray(w[:, a:b]), p=1)[0]

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(run, range(threads)))
    ref.close()
    return out


@pytest.mark.parametrize("name", ["cfg3-h2b", "cfg4-h2b", "cfg5-hss", "cfg5-h2b"])
def test_configs_full_size_column_subset(name):
    """BASELINE configs at full size and full Q. Checked against the reference library's own
    hmx::evaluate (a subset of >= 64 columns): the whole first column block
    (0-63), the seam between the first two blocks (60-67), the last 8 columns and 8 seeded
    ones, each column to <= 1e-12 relative error. Y[:,c] depends only on W[:,c]:
    a partial last column block (Q - 29) and the subset evaluated alone reproduce the full
    evaluation's columns bit for bit."""
    spec, q = config(name)
    inst = build_instance(spec)
    n = inst.cds.n
    ev = Evaluator(inst.cds)
    rng = np.random.default_rng(11)
    w = np.asfortranarray(rng.standard_normal((n, q)))
    y = ev.evaluate(w)
    cols = np.unique(np.concatenate([np.arange(0, 68), np.arange(q - 8, q), rng.choice(q, size=8, replace=False)]))
    assert len(cols) >= 64
    wsub = np.asfortranarray(w[:, cols])
    y_ref = _ref_columns(inst.cds, wsub)
    per_col = np.linalg.norm(y[:, cols] - y_ref, axis=0) / np.linalg.norm(y_ref, axis=0)
    assert per_col.max() <= TOL, (int(cols[per_col.argmax()]), float(per_col.max()))
    assert oracle.rel_frob(y[:, cols], y_ref) <= TOL
    assert np.array_equal(ev.evaluate(wsub), y[:, cols])
    qp = q - 29  # partial last column block
    assert np.array_equal(ev.evaluate(np.asfortranarray(w[:, :qp])), y[:, :qp])
    # linearity at full size on two columns
    y2 = ev.evaluate(np.asfortranarray(np.stack([w[:, cols[0]] * 3.0 + w[:, cols[1]], w[:, cols[1]]], axis=1)))
    assert oracle.rel_frob(y2[:, 0], 3.0 * y[:, cols[0]] + y[:, cols[1]]) <= TOL
    ev.close()
    inst.close()


def test_non_finite_w():
    """W with NaN and +-inf entries (the reference's GEMMs, dense.cpp:13-66, turn 0 * inf into
    NaN). Pinned semantics: columns of W that are finite give the same bits
    as without the non-finite columns (column independence holds for non-finite data too);
    in a column with a non-finite entry, Y is non-finite wherever the reference's Y is, and
    the B200 never makes an entry non-finite that the reference keeps finite. Values may
    differ in kind (+-inf on the B200 where the reference has NaN): the bases' identity
    rows are copies here, so their exact zeros never multiply an inf."""
    spec, _ = config("cfg1-hss")
    inst = build_instance(spec)
    n = inst.cds.n
    w = _w(n, 12, 77)
    rng = np.random.default_rng(5)
    bad_cols = [1, 4, 7, 10]
    for c, val in zip(bad_cols, [np.nan, np.inf, -np.inf, np.nan]):
        w[rng.integers(n), c] = val
    w[rng.integers(n), 10] = np.inf
    ev = Evaluator(inst.cds)
    y = ev.evaluate(w)
    y_ref = _ref_columns(inst.cds, w, threads=4)
    good = [c for c in range(12) if c not in bad_cols]
    clean = ev.evaluate(np.asfortranarray(w[:, good]))
    assert np.array_equal(y[:, good], clean)
    assert oracle.rel_frob(y[:, good], y_ref[:, good]) <= TOL
    nf_gpu, nf_ref = ~np.isfinite(y[:, bad_cols]), ~np.isfinite(y_ref[:, bad_cols])
    assert not np.any(nf_gpu & ~nf_ref)  # nothing non-finite that the reference keeps finite
    assert np.array_equal(nf_gpu, nf_ref), (int(nf_gpu.sum()), int(nf_ref.sum()))
    ev.close()


@pytest.mark.parametrize("name,q", [("cfg1-hss", 64), ("cfg2-h2b", 200), ("cfg5-hss", 130)])
def test_dag_launch_equals_level_launches(name, q):
    """The whole-evaluation DAG launch (default) and the level-by-level launch sequence
    compute every tile identically: bit-identical Y."""
    spec, _ = config(name)
    inst = build_instance(spec)
    ev = Evaluator(inst.cds)
    w = _w(inst.cds.n, q, 21)
    a = ev.evaluate(w)
    b = ev.evaluate(w, levels=True)
    assert np.array_equal(a, b)
    assert oracle.rel_frob(a, oracle.oracle_evaluate(inst.cds, w)) <= TOL


@pytest.mark.parametrize("q", [1, 7, 63, 65, 129, 257, 320])
def test_ragged_column_counts(q):
    """Every column count, one to several column blocks, partial last
    blocks included: the oracle's result, and the DAG equal to the level launches."""
    inst = build_instance(InstanceSpec(n=3000, d=3, leaf=48, max_rank=40, mode="tau", tau=0.7, seed=12))
    ev = Evaluator(inst.cds)
    w = _w(inst.cds.n, q, 5)
    y = ev.evaluate(w)
    assert oracle.rel_frob(y, oracle.oracle_evaluate(inst.cds, w)) <= TOL
    assert np.array_equal(y, ev.evaluate(w, levels=True))
    ev.close()
    inst.close()


@pytest.mark.parametrize("n,leaf", [(40, 16), (129, 64), (2, 1)])
def test_tiny_trees(n, leaf):
    """Two-level and single-point-leaf trees (structure.cpp:35-36 rejects one-node trees)."""
    inst = build_instance(InstanceSpec(n=n, d=2, leaf=leaf, max_rank=8, seed=3))
    w = _w(n, 5, 2)
    y = evaluate(inst.cds, EvalPlan(), w)
    assert oracle.rel_frob(y, oracle.oracle_evaluate(inst.cds, w)) <= TOL
    inst.close()


@pytest.mark.parametrize("devices", [(0,), (0, 0)])
def test_strided_w_and_y(devices):
    """Leading dimensions larger than n (odd ones included) on the host-pointer path (one
    device and two column shards) and the device-pointer path: the same bits as compact
    buffers, and the rows of Y past n are left untouched."""
    import torch

    inst = build_instance(InstanceSpec(n=3000, d=3, leaf=48, max_rank=40, mode="tau", tau=0.7, seed=12))
    n, q = inst.cds.n, 70
    ev = Evaluator(inst.cds, devices=devices)
    w = _w(n, q, 31)
    y_ref = ev.evaluate(w)
    ldw, ldy = n + 5, n + 3
    wbig = np.asfortranarray(np.full((ldw, q), np.nan))
    wbig[:n] = w
    ybig = np.asfortranarray(np.full((ldy, q), -7.0))
    ev.evaluate_host_ptr(wbig.ctypes.data, ybig.ctypes.data, q, ldw=ldw, ldy=ldy)
    assert np.array_equal(ybig[:n], y_ref)
    assert np.all(ybig[n:] == -7.0)
    if len(devices) == 1:
        wd = torch.from_numpy(wbig.T.copy()).cuda()  # (q, ldw) row major == ldw x q column major
        yd = torch.full((q, ldy), -7.0, dtype=torch.float64, device="cuda")
        ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, ldw=ldw, ldy=ldy, stream=torch_stream())
        torch.cuda.synchronize()
        yh = yd.cpu().numpy().T
        assert np.array_equal(yh[:n], y_ref)
        assert np.all(yh[n:] == -7.0)
    ev.close()
    inst.close()


def test_acceptance_criterion_3_on_the_gpu():
    """Acceptance criterion 3 (proj/tests/acceptance.cpp:125-155) with the B200 evaluator:
    50 reference-built instances (d cycling 2, 8, 32; n drawn in [256, 4096) or [256, 2048)
    for d = 32; HSS and tau = 0.65 alternating; leaf 64, rank 32, budget 64, k-NN 8,
    bacc 1e-3, seed 100 + i), W 3 columns, against the reference's evaluate_reference, for
    several plans (schedule switches the evaluator accepts): worst relative error <= 1e-13."""
    import random

    rng = random.Random(33)
    worst = 0.0
    plans = [EvalPlan(), EvalPlan(block_lowering_near=True, block_lowering_far=True, coarsen_lowering=True, peel_top=True, p=4)]
    for i in range(50):
        d = (2, 8, 32)[i % 3]
        n_max = 2048 if d == 32 else 4096
        n = 256 + rng.randrange(n_max - 255)
        spec = oracle.RefInstanceSpec(n=n, d=d, leaf=64, max_rank=32, budget=64, knn_k=8, bacc=1e-3, seed=100 + i,
                                      mode=0 if i % 2 else 1, tau=0.65 if i % 2 else 0.0)
        ri = oracle.RefInstance(spec)
        w = oracle.random_matrix(n, 3, spec.seed)
        ref = ri.evaluate_reference(w)
        for plan in plans:
            worst = max(worst, oracle.rel_frob(evaluate(ri.cds, plan, w), ref))
    assert worst <= 1e-13, worst


@pytest.mark.parametrize("devices", [(0,), (0, 0)])
def test_pinned_and_pageable_host_paths_agree(devices):
    """The host-pointer path runs the copy-engine pipeline on pinned buffers and the pinned
    bounce path on pageable ones (numpy): the same bits, on one device and on two column
    shards, and equal to the device-pointer path."""
    import torch

    spec, _ = config("cfg2-h2b")
    inst = build_instance(spec)
    n, q = inst.cds.n, 200
    ev = Evaluator(inst.cds, devices=devices)
    w = _w(n, q, 41)
    y_pageable = ev.evaluate(w)
    wh = torch.from_numpy(w.T.copy()).pin_memory()
    yh = torch.empty_like(wh).pin_memory()
    ev.evaluate_host_ptr(wh.data_ptr(), yh.data_ptr(), q)
    assert np.array_equal(yh.numpy().T, y_pageable)
    if len(devices) == 1:
        wd = wh.cuda()
        yd = torch.empty_like(wd)
        ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=torch_stream())
        torch.cuda.synchronize()
        assert np.array_equal(yd.cpu().numpy().T, y_pageable)
    ev.close()
    inst.close()


@pytest.mark.parametrize("name,q", [("cfg1-hss", 64), ("cfg1-hss", 150), ("cfg2-h2b", 96)])
def test_fused_small_problem_launch_equals_three_launches(name, q, monkeypatch):
    """Small problems run one launch: the permutations inside eval_dag (Wp gathered per
    (leaf, column block), final leaf rows stored straight into Y). The same evaluation with
    the separate permute kernels (HMXG_NO_FUSED) gives the same bits, on the host-pointer
    and the device-pointer paths, and both match the oracle."""
    import torch

    spec, _ = config(name)
    inst = build_instance(spec)
    n = inst.cds.n
    ev = Evaluator(inst.cds)
    w = _w(n, q, 17)
    fused = ev.evaluate(w)
    assert ev.info().launches_per_eval == 1
    wd = torch.from_numpy(w.T.copy()).cuda()
    yd = torch.empty_like(wd)
    ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=torch_stream(), graph=False, sync=True)
    assert np.array_equal(yd.cpu().numpy().T, fused)
    monkeypatch.setenv("HMXG_NO_FUSED", "1")
    three = ev.evaluate(w)
    assert ev.info().launches_per_eval == 3
    ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=torch_stream(), graph=False, sync=True)
    assert np.array_equal(yd.cpu().numpy().T, three)
    monkeypatch.delenv("HMXG_NO_FUSED")
    assert np.array_equal(fused, three)
    assert np.array_equal(ev.evaluate(w), fused)  # counters left clean by either launch sequence
    assert oracle.rel_frob(fused, oracle.oracle_evaluate(inst.cds, w)) <= TOL
    ev.close()


@pytest.mark.parametrize("name,q", [("cfg1-hss", 64), ("cfg1-hss", 37), ("tiny", 9), ("ragged", 100)])
def test_ctree_mode_gives_the_dag_bits(name, q, monkeypatch):
    """CTree mode (HMXG_CTREE=1, MatRox's coarsened sub-tree execution: every task but the near
    field runs inside one CTA cluster per 8-column octet, levels separated by cluster barriers)
    runs each 8 x 8 fragment's exact DMMA sequence of the DAG: the same bits as the DAG launch
    and the level launches, through the host and the device paths, for 2, 4 and 8-CTA clusters."""
    import torch

    monkeypatch.setenv("HMXG_NO_FLAT", "1")  # CTree runs the level-by-level tree
    if name == "tiny":
        inst = build_instance(InstanceSpec(n=129, d=3, leaf=16, max_rank=12, seed=3))
    elif name == "ragged":
        inst = build_instance(InstanceSpec(n=1500, d=5, leaf=40, max_rank=24, mode="budget", budget=0.1, seed=9,
                                           kernel="exponential", h=1.5))
    else:
        inst = build_instance(config(name)[0])
    n = inst.cds.n
    ev = Evaluator(inst.cds)
    w = _w(n, q, 23)
    dag = ev.evaluate(w)
    lev = ev.evaluate(w, levels=True)
    assert np.array_equal(dag, lev)
    monkeypatch.setenv("HMXG_CTREE", "1")
    wd = torch.from_numpy(w.T.copy()).cuda()
    yd = torch.empty_like(wd)
    for cs in ("2", "4", "8"):
        monkeypatch.setenv("HMXG_CT_CLUSTER", cs)
        assert np.array_equal(ev.evaluate(w), dag), cs
        yd.fill_(np.nan)
        ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), q, stream=torch_stream(), graph=False, sync=True)
        assert np.array_equal(yd.cpu().numpy().T, dag), cs
    assert np.array_equal(ev.evaluate(w, levels=True), dag)
    monkeypatch.delenv("HMXG_CTREE")
    assert np.array_equal(ev.evaluate(w), dag)  # counters and item lists clean after the mode switch
    assert oracle.rel_frob(dag, oracle.oracle_evaluate(inst.cds, w)) <= TOL
    ev.close()
    inst.close()


@pytest.mark.parametrize("name", ["cfg1-hss", "small", "uneven"])
def test_flat_tree(name, monkeypatch):
    """The flat tree of small trees (DESIGN.md kernel 6: the internal upward and far+downward
    levels replaced by composite transfer products formed at upload) agrees with the level-by-
    level tree (HMXG_NO_FLAT=1) to rounding and with the oracle; it is plan-wide, so a column
    computed alone, in a 7-column shard or in the full block gives the same bits, and the DAG
    equals the level launches bit for bit."""
    if name == "small":  # (flat-eligible: n <= 65536, <= 1024 nodes, composites cheap)
        inst = build_instance(InstanceSpec(n=2048, d=3, leaf=64, max_rank=32, seed=8, h=0.5))
    elif name == "uneven":  # two-means tree, 3000 points: leaves of different sizes
        inst = build_instance(InstanceSpec(n=3000, d=2, leaf=128, max_rank=40, seed=3, h=1.0, split="twomeans"))
    else:
        inst = build_instance(config(name)[0])
    n, q = inst.cds.n, 64
    w = _w(n, q, 29)
    ev = Evaluator(inst.cds)
    y = ev.evaluate(w)
    assert np.array_equal(ev.evaluate(w, levels=True), y)
    for c0, c1 in [(5, 6), (10, 17), (63, 64)]:
        assert np.array_equal(ev.evaluate(np.asfortranarray(w[:, c0:c1])), y[:, c0:c1])
    monkeypatch.setenv("HMXG_NO_FLAT", "1")
    ev_levels = Evaluator(inst.cds)
    y_levels = ev_levels.evaluate(w)
    assert oracle.rel_frob(y, y_levels) <= 1e-13
    assert oracle.rel_frob(y, oracle.oracle_evaluate(inst.cds, w)) <= TOL
    ev.close()
    ev_levels.close()
    inst.close()


@pytest.mark.parametrize("name,q", [("cfg2-h2b", 200), ("hss", 320)])
def test_subtree_pipelined_order_gives_the_same_bits(name, q, monkeypatch):
    """Wide DAGs claim their work items in a subtree-pipelined order (the far+downward levels
    of one group of subtrees interleaved with the previous group's leaf rows, hmxg.cu
    pipe_depth). Only the order changes: the same bits as the level-major order (HMXG_PIPE=0)
    for every grouping depth, and the oracle's result."""
    monkeypatch.setenv("HMXG_NO_FLAT", "1")
    monkeypatch.setenv("HMXG_SPLIT_FRAC", "0")  # (the pipelined order runs the combined leaf tasks)
    if name == "hss":
        inst = build_instance(InstanceSpec(n=32768, d=3, leaf=64, max_rank=48, h=0.2, tol=1e-6, seed=6))
    else:
        inst = build_instance(config(name)[0])
    w = _w(inst.cds.n, q, 31)
    monkeypatch.setenv("HMXG_PIPE", "0")
    ev = Evaluator(inst.cds)
    base = ev.evaluate(w)
    ev.close()
    monkeypatch.setenv("HMXG_PIPE_MIN", "0")
    for d0 in ("1", "2", "4"):
        monkeypatch.setenv("HMXG_PIPE", d0)
        ev = Evaluator(inst.cds)
        assert np.array_equal(ev.evaluate(w), base), d0
        assert np.array_equal(ev.evaluate(w, levels=True), base), d0
        ev.close()
    assert oracle.rel_frob(base, oracle.oracle_evaluate(inst.cds, w)) <= TOL
    inst.close()
