"""Worker of tests/test_gpu_multirank.py, launched by torchrun with 2 ranks on one GPU over
gloo (the ranks' kernels never wait on each other: every exchange is between launches).

    multirank_worker.py MODE OUTDIR   MODE: split | replicated
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1812_07152_b200 import Context, Evaluator, InstanceSpec, build_instance  # noqa: E402
from paper_1812_07152_b200.distributed import TorchComm, column_shard, gather_columns  # noqa: E402

SPEC = InstanceSpec(n=9000, d=3, leaf=64, max_rank=48, mode="budget", budget=0.05, h=0.3, seed=21)
Q = 150


def main():
    mode, out = sys.argv[1], sys.argv[2]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    inst = build_instance(SPEC)
    w = np.asfortranarray(np.random.default_rng(3).standard_normal((inst.cds.n, Q)))
    comm = TorchComm(hbm_budget=1 if mode == "split" else 0)
    ctx = Context((0,), comm=comm)
    ev = Evaluator(inst.cds, context=ctx)
    info = ev.info()
    if mode == "split":
        y = ev.evaluate(w)  # collective: the same full W on every rank, the full Y back
    else:
        c0, c1 = column_shard(Q, world, rank)
        y = gather_columns(ev.evaluate(np.asfortranarray(w[:, c0:c1])), Q)
    np.savez(os.path.join(out, f"rank{rank}.npz"), y=y, split_parts=info.split_parts, part=info.part,
             device_bytes=info.device_bytes, errors=np.array(comm.errors, dtype=object), allow_pickle=True)
    ev.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
