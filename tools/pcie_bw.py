"""Pinned host<->device copy bandwidth on the box: each direction alone and both at once (dev tool)."""
import torch

GB = 1 << 30
n = 2 * GB // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, by in [("h2d", h2d, 2 * GB), ("d2h", d2h, 2 * GB), ("both", both, 4 * GB)]:
    fn()
    t = timed(fn)
    print(f"{name}: {by / t / 1e9:.1f} GB/s ({t * 1e3:.1f} ms)")
for chunk_mb in (16, 64, 128, 512):
    m = chunk_mb * (1 << 20) // 8
    def chunked():
        for k in range(0, n, m):
            with torch.cuda.stream(s1):
                d_in[k:k + m].copy_(h_in[k:k + m], non_blocking=True)
            with torch.cuda.stream(s2):
                h_out[k:k + m].copy_(d_out[k:k + m], non_blocking=True)
    t = timed(chunked)
    print(f"both chunked {chunk_mb} MB: {4 * GB / t / 1e9:.1f} GB/s")
