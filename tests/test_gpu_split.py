"""Subtree-split fallback for a CDS larger than one GPU: each part holds only
its own subtrees' generators, the parts exchange the skeleton weights T between two stages
and sum their Y. The result must equal the single-device evaluation bit for bit (every
tile is computed identically; the exchanges add exact zeros)."""
import os

import numpy as np
import pytest

import oracle
from paper_1812_07152_b200 import Evaluator, InstanceSpec, build_instance, config
from paper_1812_07152_b200.distributed import SplitPart, split_evaluate
from paper_1812_07152_b200.executor import torch_stream

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,nparts,q", [("cfg1-hss", 2, 64), ("cfg2-h2b", 3, 70), ("cfg2-h2b", 4, 128)])
def test_split_parts_equal_single_device(name, nparts, q, monkeypatch):
    """(The split runs the level-by-level tree; the single-device reference here does too:
    small trees otherwise run the flat tree, equal to rounding, checked at the end.)"""
    import torch

    monkeypatch.setenv("HMXG_NO_FLAT", "1")
    spec, _ = config(name)
    inst = build_instance(spec)
    n = inst.cds.n
    w = torch.randn((q, n), dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    parts = [SplitPart(inst.cds, nparts, k) for k in range(nparts)]
    y = split_evaluate(inst.cds, w, parts=parts)
    ev = Evaluator(inst.cds)
    y_full = torch.empty_like(w)
    ev.evaluate_device(w.data_ptr(), y_full.data_ptr(), q, sync=True, stream=torch_stream())
    assert torch.equal(y, y_full)
    yn = y.cpu().numpy().T
    assert oracle.rel_frob(yn, oracle.oracle_evaluate(inst.cds, w.cpu().numpy().T)) <= 1e-12
    # each part holds only its share of the generators (plus the replicated top levels)
    full_bytes = ev.info().device_bytes
    part_bytes = [p.info().device_bytes for p in parts]
    assert max(part_bytes) < full_bytes
    for p in parts:
        p.close()
    monkeypatch.delenv("HMXG_NO_FLAT")
    ev_flat = Evaluator(inst.cds)  # the default replicated upload (flat tree for small trees)
    y_flat = torch.empty_like(w)
    ev_flat.evaluate_device(w.data_ptr(), y_flat.data_ptr(), q, sync=True, stream=torch_stream())
    assert oracle.rel_frob(y_flat.cpu().numpy().T, yn) <= 1e-13


def test_split_tau_instance_and_reference():
    import torch

    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=3000, d=3, mode=0, tau=0.65, leaf=64, max_rank=32, seed=7))
    n, q = ri.cds.n, 9
    wn = oracle.random_matrix(n, q, 4)
    w = torch.from_numpy(np.ascontiguousarray(wn.T)).cuda()
    y = split_evaluate(ri.cds, w, nparts=2).cpu().numpy().T
    assert oracle.rel_frob(y, ri.evaluate(wn)) <= 1e-12


def _rank(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_1812_07152_b200 import build_instance, config
    from paper_1812_07152_b200.distributed import SplitPart, split_evaluate

    import datetime

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # both ranks share GPU 0 in this test
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    spec, _ = config("cfg2-h2b")
    inst = build_instance(spec)
    w = torch.randn((40, inst.cds.n), dtype=torch.float64, device="cuda",
                    generator=torch.Generator("cuda").manual_seed(5))
    y = split_evaluate(inst.cds, w, parts=[SplitPart(inst.cds, world, rank)])
    if rank == 0:
        np.save(os.path.join(out_dir, "y.npy"), y.cpu().numpy())
        np.save(os.path.join(out_dir, "w.npy"), w.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_split_two_ranks_exchange(tmp_path):
    from conftest import spawn_bounded

    spawn_bounded(_rank, (2, None, str(tmp_path)), nprocs=2, deadline_s=400.0)
    spec, _ = config("cfg2-h2b")
    inst = build_instance(spec)
    w = np.load(tmp_path / "w.npy")
    y_full = Evaluator(inst.cds).evaluate(np.asfortranarray(w.T))
    assert np.array_equal(np.load(tmp_path / "y.npy").T, y_full)
