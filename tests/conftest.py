import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box with -m gpu)")
    config.addinivalue_line("markers", "slow: longer CPU checks")


def _has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_bounded(fn, args, nprocs, deadline_s=150.0, attempts=2):
    """mp.spawn with a deadline: the ranks are joined in slices and killed when the deadline
    passes (a lost rendezvous would otherwise hold the whole suite); one retry on a new port.
    `args[1]` is the port slot."""
    import time

    last = None
    for _ in range(attempts):
        a = list(args)
        a[1] = free_port()
        import torch.multiprocessing as mp

        ctx = mp.start_processes(fn, args=tuple(a), nprocs=nprocs, join=False, start_method="spawn")
        t0 = time.time()
        try:
            while not ctx.join(timeout=2.0):
                if time.time() - t0 > deadline_s:
                    raise TimeoutError(f"ranks still running after {deadline_s:.0f} s")
            return
        except Exception as e:  # a rank failed, or the deadline passed
            last = e
            for pr in ctx.processes:
                if pr.is_alive():
                    pr.kill()
            for pr in ctx.processes:
                pr.join(5.0)
    raise last
