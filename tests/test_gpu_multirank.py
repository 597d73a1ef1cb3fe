"""Multi-process paths on the B200 kernels: two ranks launched by torchrun on one
GPU over gloo, every exchange between launches (the ranks' kernels never wait on each other).

* the subtree-split fallback through the C-ABI: hmxg_create_comm with an HBM budget the CDS
  exceeds, so hmxg_upload holds one subtree part per rank and hmxg_evaluate is collective
  (all-gather of the published T rows, then of the result rows): bit-identical to the
  single-device evaluation on every rank, each rank holding fewer generator bytes;
* the replicated, column-sharded path: each rank evaluates its column shard, the shards are
  all-gathered: bit-identical to the single-device evaluation;
* bench.py's N > 1 path (torchrun, gloo, both ranks on device 0): one JSON line for 2 ranks.
Tolerance against the oracle: relative Frobenius <= 1e-12."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.mark.parametrize("mode", ["split", "replicated"])
def test_two_ranks_on_the_b200_kernels(mode, tmp_path):
    import multirank_worker as mw

    from paper_1812_07152_b200 import Evaluator, build_instance

    out = _torchrun([os.path.join(ROOT, "tests", "multirank_worker.py"), mode, str(tmp_path)])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    inst = build_instance(mw.SPEC)
    w = np.asfortranarray(np.random.default_rng(3).standard_normal((inst.cds.n, mw.Q)))
    ev = Evaluator(inst.cds)
    y1 = ev.evaluate(w)
    whole = ev.info().device_bytes
    ev.close()
    assert oracle.rel_frob(y1, oracle.oracle_evaluate(inst.cds, w)) <= 1e-12
    parts = set()
    for r in range(2):
        z = np.load(tmp_path / f"rank{r}.npz", allow_pickle=True)
        assert len(z["errors"]) == 0, z["errors"]
        assert np.array_equal(z["y"], y1), f"rank {r}"
        if mode == "split":
            assert int(z["split_parts"]) == 2
            assert int(z["device_bytes"]) < whole  # each part holds only what its tiles read
            parts.add(int(z["part"]))
        else:
            assert int(z["split_parts"]) == 1
    if mode == "split":
        assert parts == {0, 1}


def test_bench_two_ranks_gloo_on_one_device():
    out = _torchrun([os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", "gloo", "--device", "0",
                     "--config", "cfg2-h2b", "--q", "128", "--steps", "2", "--warmup", "3", "--e2e-steps", "1",
                     "--dropin-steps", "0", "--extra", "", "--no-cpu-baseline"])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["config"]["q_per_gpu"] == 64 and line["config"]["q_total"] == 128
    assert np.isfinite(line["value"]) and line["value"] > 0
    assert "world=2" in out.stderr  # the process group came up with both ranks
