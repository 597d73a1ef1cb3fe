"""GPU compression vs the reference's compress on the same inputs (dev tool).

The reference instance (tst::make_instance) is built on the host, which times its own
hmx::compress (single thread, -O3); the GPU then recompresses from the same tree, samples
and points."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1812_07152_b200.accuracy import Kernel
from paper_1812_07152_b200.compress import gpu_compress

for n, d, leaf, rank, kern, h in [(16384, 3, 128, 64, 1, 1.0), (32768, 3, 128, 64, 0, 0.5), (65536, 3, 256, 128, 0, 0.2)]:
    t = time.time()
    ri = oracle.RefInstance(oracle.RefInstanceSpec(n=n, d=d, leaf=leaf, max_rank=rank, kernel=kern, h=h, seed=1,
                                                   bacc=1e-6))
    t_build = time.time() - t
    t_ref = oracle._ref_lib().hmxr_compress_seconds(ri._h)
    import ctypes as C
    rsum = C.c_uint64()
    t_bases = min(oracle._ref_lib().hmxr_bases_seconds(ri._h, C.byref(rsum)) for _ in range(2))
    sp, si = ri.samples()
    k = Kernel.inverse_distance() if kern == 1 else Kernel.gaussian(h)
    gpu_compress(ri.points(), k, ri.cds, sp, si, 1e-6, rank)  # warm-up
    ts = []
    for _ in range(3):
        t = time.time()
        b = gpu_compress(ri.points(), k, ri.cds, sp, si, 1e-6, rank)
        ts.append(time.time() - t)
    same = all(bb.srank == ri.basis(i)[0] for i, bb in enumerate(b))
    print(f"n={n} d={d} leaf={leaf} s={rank} kernel={'invdist' if kern else 'gaussian'}: reference compress "
          f"{t_ref:.3f} s (bases + far/near blocks, 1 thread); reference bases only {t_bases:.3f} s (1 thread, "
          f"sum of ranks {rsum.value}); GPU bases {min(ts):.3f} s (incl. host readback); same ranks: {same}; "
          f"bases speed-up {t_bases / min(ts):.1f}x; instance build {t_build:.1f} s", flush=True)
    ri.close()
