"""Device timing of the GPU error oracle's exact kernel products (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1812_07152_b200.accuracy import DevicePoints, Kernel, sample_rows
from paper_1812_07152_b200.executor import EvalStats

PEAK = 37.0e12
cases = [("cfg5 sampled", 262144, 3, 0.1, 256, 2048), ("dense n=16384", 16384, 3, 0.5, 16384, 64),
         ("dense n=16384 q=512", 16384, 3, 0.5, 16384, 512)]
for name, n, d, h, nr, q in cases:
    rng = np.random.default_rng(0)
    pts = rng.random((n, d))
    dp = DevicePoints(pts, Kernel.gaussian(h))
    w = torch.randn(q, n, dtype=torch.float64, device="cuda")
    y = torch.empty(q, nr, dtype=torch.float64, device="cuda")
    rows = None if nr == n else sample_rows(n, 1)
    for _ in range(2):
        dp.kernel_rows_device(rows, w.data_ptr(), y.data_ptr(), q)
    st = EvalStats()
    ms = []
    for _ in range(5):
        dp.kernel_rows_device(rows, w.data_ptr(), y.data_ptr(), q, stats=st)
        ms.append(st.device_ms)
    t = float(np.median(ms))
    fl = 2.0 * nr * n * q
    print(f"{name}: rows={nr} n={n} q={q} {t:.3f} ms {fl/t/1e9:.2f} TFLOP/s ({fl/t/1e9/37.0*100:.1f}% of FP64 peak) "
          f"launches={st.launches}", flush=True)
    dp.close()
