"""world_size-2 gloo test of the column-sharded N>1 path (CPU).

Each rank builds the same CDS, checks the replication fingerprint, evaluates its column
shard (the oracle restatement stands in for the B200 kernels here: this is a host-logic
test), and the all-gathered shards must equal the full single-process result bit for bit
(column independence). The max-over-ranks timing reduction is checked too.
"""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp


from conftest import spawn_bounded as _spawn_bounded  # noqa: E402


def _worker(rank, world, port, q, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import oracle
    from paper_1812_07152_b200 import InstanceSpec, build_instance
    from paper_1812_07152_b200.distributed import (check_replicated, column_shard, gather_columns,
                                                   max_over_ranks)

    import datetime

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # a bounded rendezvous: the port was free a moment ago, but nothing holds it until rank 0
    # binds it (the default store timeout is half an hour)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    inst = build_instance(InstanceSpec(n=3000, d=3, leaf=64, max_rank=32, mode="budget", budget=0.1, seed=9,
                                       threads=2))
    check_replicated(inst.cds)
    w = np.asfortranarray(np.random.default_rng(5).standard_normal((inst.cds.n, q)))
    c0, c1 = column_shard(q, world, rank)
    y_local = oracle.oracle_evaluate(inst.cds, w[:, c0:c1])
    y = gather_columns(y_local, q)
    t = max_over_ranks(1.0 + rank)
    if rank == 0:
        np.save(os.path.join(out_dir, "y.npy"), y)
        np.save(os.path.join(out_dir, "t.npy"), np.array([t]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("q", [7, 16])
def test_column_sharded_gloo_world2(tmp_path, q):
    _spawn_bounded(_worker, (2, None, q, str(tmp_path)), nprocs=2)
    import oracle
    from paper_1812_07152_b200 import InstanceSpec, build_instance

    inst = build_instance(InstanceSpec(n=3000, d=3, leaf=64, max_rank=32, mode="budget", budget=0.1, seed=9))
    w = np.asfortranarray(np.random.default_rng(5).standard_normal((inst.cds.n, q)))
    full = oracle.oracle_evaluate(inst.cds, w)
    assert np.array_equal(np.load(tmp_path / "y.npy"), full)
    assert float(np.load(tmp_path / "t.npy")[0]) == 2.0


def test_column_shard_partition():
    from paper_1812_07152_b200.distributed import column_shard

    for q in (0, 1, 5, 2048, 2049):
        for world in (1, 2, 3, 8):
            cuts = [column_shard(q, world, r) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == q
            assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
            assert max(c1 - c0 for c0, c1 in cuts) - min(c1 - c0 for c0, c1 in cuts) <= 1
