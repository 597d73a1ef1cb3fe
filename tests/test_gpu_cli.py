"""`hmx eval` on the B200 (GPU): a CDS the reference wrote (hmat.cds) is read by the
native mmap reader, evaluated through the CUDA path and compared with the reference's
own hmx::evaluate on its own CDS (rel. Frobenius <= 1e-12, BASELINE north_star)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1812_07152_b200 import cli
from paper_1812_07152_b200.serial import load_matrix, random_w

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def stored(tmp_path_factory):
    d = tmp_path_factory.mktemp("art")
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=3000, d=3, mode=0, tau=0.65, leaf=64, max_rank=48, seed=9))
    ri.save_cds(str(d / "hmat.cds"))
    return d, ri


def test_cli_eval_w_file(stored, capsys):
    d, ri = stored
    w = oracle.random_matrix(3000, 37, 4)
    oracle.ref_save_matrix(str(d / "w.bin"), w)
    rc = cli.main(["eval", "--out", str(d), "--w", str(d / "w.bin"), "--y", str(d / "y.bin")])
    assert rc == 0
    assert "eval: n=3000 q=37" in capsys.readouterr().out
    y = oracle.ref_load_matrix(str(d / "y.bin"))
    assert oracle.rel_frob(y, ri.evaluate(w)) <= 1e-12


def test_cli_eval_random_w(stored):
    d, ri = stored
    rc = cli.main(["eval", "--out", str(d), "--q", "16", "--seed", "3", "--y", str(d / "y2.bin")])
    assert rc == 0
    y = load_matrix(str(d / "y2.bin"))
    assert oracle.rel_frob(y, ri.evaluate(random_w(3000, 16, 3))) <= 1e-12


def test_cli_eval_subprocess(stored):
    d, ri = stored
    r = subprocess.run([sys.executable, "-m", "paper_1812_07152_b200", "eval", "--out", str(d), "--q", "5",
                        "--seed", "1", "--y", str(d / "y3.bin")], cwd=ROOT, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert "locked_pairs=0" in r.stdout
    y = load_matrix(str(d / "y3.bin"))
    assert oracle.rel_frob(y, ri.evaluate(random_w(3000, 5, 1))) <= 1e-12


def test_cli_eval_row_mismatch(stored):
    d, _ = stored
    oracle.ref_save_matrix(str(d / "wbad.bin"), np.ones((10, 2)))
    assert cli.main(["eval", "--out", str(d), "--w", str(d / "wbad.bin")]) == cli.EXIT_USAGE


def test_cli_accuracy_sweep(tmp_path, capsys):
    rc = cli.main(["accuracy", "--synth", "uniform", "--n", "4096", "--d", "3", "--leaf", "128", "--max-rank", "64",
                   "--kernel", "gaussian:0.5", "--bacc-list", "1e-2", "1e-5", "--q", "8", "--seed", "2"])
    assert rc == 0
    out = capsys.readouterr().out.splitlines()
    i = out.index("bacc,eps_f,eval_seconds,p2_seconds")
    rows = [line.split(",") for line in out[i + 1:i + 3]]
    eps = [float(r[1]) for r in rows]
    assert 0.0 < eps[1] < eps[0] < 1.0  # a tighter tolerance gives a smaller error
    assert out[i + 3].startswith("# p1=")
