"""The reference's on-disk formats (CPU): hmat.cds, matrix files, plan.json, the CLI's
random W, and the CLI's error behaviour.

* ``load_cds`` (native mmap reader, include/hmxg.h hmxg_cds_file_open) reads a file the
  reference wrote with hmx::save_cds (serial.cpp:271-277) into exactly the reference's
  own CDS arrays, bit for bit.
* ``save_cds`` writes a file hmx::load_cds (serial.cpp:299-308) accepts, and the reference
  evaluates the loaded CDS to the same bits as the in-memory one.
* Matrix files round-trip both ways with hmx::save_matrix / hmx::load_matrix.
* Malformed files are refused like the reference refuses them (io_error -> exit 3).
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1812_07152_b200 import InstanceSpec, build_instance, cli
from paper_1812_07152_b200.serial import (CdsFile, IoError, load_cds, load_matrix, load_plan, random_w, save_cds,
                                          save_matrix)

needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")

ARRAYS = ("parent", "lchild", "rchild", "start", "end", "level", "perm", "sranks", "participating", "near_pairs",
          "far_pairs", "v_order", "dptr", "bptr", "vptr", "dgen", "bgen", "vgen")


def assert_same_cds(a, b):
    assert (a.n, a.num_nodes, a.height) == (b.n, b.num_nodes, b.height)
    for name in ARRAYS:
        x, y = getattr(a, name), getattr(b, name)
        assert x.dtype == y.dtype and x.shape == y.shape, name
        assert np.array_equal(x, y), name


@needs_ref
@pytest.mark.parametrize("n,d,mode,tau,leaf,rank,seed", [
    (512, 2, 1, 0.0, 64, 64, 1), (380, 8, 0, 0.65, 16, 24, 2), (1024, 3, 0, 0.65, 64, 32, 7),
])
def test_reader_matches_reference_cds(tmp_path, n, d, mode, tau, leaf, rank, seed):
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=n, d=d, mode=mode, tau=tau, leaf=leaf, max_rank=rank, seed=seed,
                                                   p=4, agg=2))
    path = str(tmp_path / "hmat.cds")
    ri.save_cds(path)
    f = CdsFile(path)
    assert_same_cds(f.cds, ri.cds)
    assert f.dim == d and f.max_rank == rank and f.bacc == ri.spec.bacc
    # the reference's own reader sees the same CDS
    rc = oracle.RefCds.load(path)
    assert_same_cds(rc.cds, ri.cds)
    f.close()


@needs_ref
@pytest.mark.parametrize("mode", ["hss", "budget", "tau"])
def test_writer_is_read_by_reference(tmp_path, mode):
    inst = build_instance(InstanceSpec(n=1500, d=3, leaf=48, max_rank=24, mode=mode, seed=11))
    path = str(tmp_path / "hmat.cds")
    save_cds(path, inst.cds, dim=3, bacc=1e-5, max_rank=24)
    rc = oracle.RefCds.load(path)
    assert_same_cds(rc.cds, inst.cds)
    assert_same_cds(load_cds(path), inst.cds)
    # the reference evaluates the loaded CDS to the same bits as the oracle on the original
    w = oracle.random_matrix(inst.cds.n, 3, 5)
    y_ref, _ = rc.evaluate(w)
    assert np.array_equal(y_ref, oracle.oracle_evaluate(inst.cds, w))
    inst.close()


def test_reader_rejects_malformed(tmp_path):
    inst = build_instance(InstanceSpec(n=600, d=2, leaf=32, max_rank=16, seed=3))
    path = str(tmp_path / "hmat.cds")
    save_cds(path, inst.cds)
    blob = open(path, "rb").read()
    bad = tmp_path / "bad.cds"
    cases = {
        "bad tag": b"XDS1" + blob[4:],
        "version": blob[:4] + (2).to_bytes(4, "little") + blob[8:],
        "truncated": blob[: len(blob) // 2],
        "tiny": blob[:6],
        "header/tree": blob[:8] + (inst.cds.n + 1).to_bytes(8, "little") + blob[16:],
    }
    for what, data in cases.items():
        bad.write_bytes(data)
        with pytest.raises(IoError):
            load_cds(str(bad))
    with pytest.raises(IoError):
        load_cds(str(tmp_path / "missing.cds"))
    # trailing bytes are ignored, as by hmx::load_cds
    bad.write_bytes(blob + b"\0" * 8)
    assert_same_cds(load_cds(str(bad)), inst.cds)
    inst.close()


@needs_ref
def test_matrix_files_roundtrip_with_reference(tmp_path):
    rng = np.random.default_rng(0)
    for shape in [(7, 3), (1, 1), (5, 0), (300, 17)]:
        m = np.asfortranarray(rng.standard_normal(shape))
        p1, p2 = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
        oracle.ref_save_matrix(p1, m)
        assert np.array_equal(load_matrix(p1), m)
        save_matrix(p2, m)
        assert open(p1, "rb").read() == open(p2, "rb").read()
        assert np.array_equal(oracle.ref_load_matrix(p2), m)


def test_matrix_file_errors(tmp_path):
    p = tmp_path / "m.bin"
    save_matrix(str(p), np.ones((4, 2)))
    blob = p.read_bytes()
    p.write_bytes(blob + b"x")
    with pytest.raises(IoError, match="trailing"):
        load_matrix(str(p))
    p.write_bytes(blob[:-1])
    with pytest.raises(IoError):
        load_matrix(str(p))
    with pytest.raises(IoError):
        load_matrix(str(tmp_path / "none.bin"))


@needs_ref
@pytest.mark.parametrize("n,q,seed", [(100, 3, 0), (513, 17, 42), (1, 1, 2**64 - 1)])
def test_cli_random_w_matches_reference_rng(n, q, seed):
    assert np.array_equal(random_w(n, q, seed), oracle.ref_cli_random_w(n, q, seed))


def test_plan_json(tmp_path):
    p = tmp_path / "plan.json"
    p.write_text(json.dumps({"block_lowering_near": True, "block_lowering_far": False, "coarsen_lowering": True,
                             "peel_top": False, "p": 12, "block_threshold": 64, "coarsen_threshold": 4}))
    plan = load_plan(str(p))
    assert plan.p == 12 and plan.block_lowering_near and plan.coarsen_lowering and plan.block_threshold == 64
    p.write_text("{\"p\": 1}")
    with pytest.raises(IoError):
        load_plan(str(p))


def test_cli_exit_codes(tmp_path, capsys):
    assert cli.main(["eval", "--out", str(tmp_path / "nowhere")]) == cli.EXIT_IO
    assert cli.main(["eval", "--bogus"]) == cli.EXIT_USAGE
    assert cli.main([]) == cli.EXIT_USAGE
    assert cli.main(["inspect", "--mode", "weird", "--out", str(tmp_path)]) == cli.EXIT_USAGE


@needs_ref
def test_cli_inspect_writes_reference_readable_cds(tmp_path, capsys):
    out = str(tmp_path / "art")
    rc = cli.main(["inspect", "--synth", "uniform", "--n", "2000", "--d", "3", "--leaf", "64", "--max-rank", "32",
                   "--kernel", "gaussian:0.5", "--seed", "7", "--out", out])
    assert rc == 0
    text = capsys.readouterr().out
    assert "config: cmd=inspect n=2000 d=3" in text and "p2: max_srank=" in text
    ref = oracle.RefCds.load(os.path.join(out, "hmat.cds"))
    assert_same_cds(ref.cds, load_cds(os.path.join(out, "hmat.cds")))
    assert load_plan(os.path.join(out, "plan.json")).coarsen_threshold == 4
