import os, sys, time
sys.path.insert(0, '/root/repo')
import oracle
from paper_1812_07152_b200.accuracy import Kernel
from paper_1812_07152_b200.compress import gpu_compress
ri = oracle.RefInstance(oracle.RefInstanceSpec(n=65536, d=3, leaf=256, max_rank=128, kernel=0, h=0.2, seed=1, bacc=1e-6))
sp, si = ri.samples()
gpu_compress(ri.points(), Kernel.gaussian(0.2), ri.cds, sp, si, 1e-6, 128)
os.environ['HMXG_COMPRESS_TRACE'] = '1'
t = time.time(); gpu_compress(ri.points(), Kernel.gaussian(0.2), ri.cds, sp, si, 1e-6, 128); print('total', time.time() - t)
