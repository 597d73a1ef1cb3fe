import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, psutil
import oracle
from paper_1812_07152_b200 import Evaluator, InstanceSpec, build_instance
from paper_1812_07152_b200.accuracy import Kernel, DevicePoints
from paper_1812_07152_b200.distributed import split_evaluate
from paper_1812_07152_b200.compress import gpu_compress
from paper_1812_07152_b200.executor import torch_stream
proc = psutil.Process()
def stat(tag):
    free, tot = torch.cuda.mem_get_info()
    print(f"{tag:28s} gpu used {(tot-free)/2**20:9.1f} MiB  rss {proc.memory_info().rss/2**20:9.1f} MiB  fds {proc.num_fds()} threads {proc.num_threads()}", flush=True)
spec = InstanceSpec(n=3000, d=3, leaf=64, max_rank=32, seed=5, h=0.5)
inst = build_instance(spec)
w = np.asfortranarray(np.random.default_rng(1).standard_normal((3000, 70)))
wd = torch.from_numpy(w.T.copy()).cuda()
stat("start")
for rep in range(3):
    for _ in range(200):
        ev = Evaluator(inst.cds); ev.evaluate(w); ev.close()
    stat(f"200 x Evaluator host eval")
for rep in range(2):
    for _ in range(200):
        ev = Evaluator(inst.cds); yd = torch.empty_like(wd)
        ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), 70, stream=torch_stream(), graph=True, sync=True)
        ev.evaluate_device(wd.data_ptr(), yd.data_ptr(), 70, stream=torch_stream(), graph=True, sync=True); ev.close()
    stat("200 x device graph eval")
for rep in range(2):
    for _ in range(100):
        two = Evaluator(inst.cds, devices=(0, 0)); two.evaluate(w); two.close()
    stat("100 x two shards")
import os as _os
_os.environ["HMXG_NO_FLAT"] = "1"
for rep in range(2):
    for _ in range(100):
        split_evaluate(inst.cds, wd, nparts=2)
    stat("100 x split_evaluate")
del _os.environ["HMXG_NO_FLAT"]
spec2 = InstanceSpec(n=3000, d=3, leaf=64, max_rank=32, seed=5, h=0.5, skip_near=True)
lean = build_instance(spec2)
for rep in range(2):
    for _ in range(100):
        ev = Evaluator(lean.cds, points=lean.points(), kernel=Kernel("gaussian", 0.5), near_on_the_fly=True); ev.evaluate(w); ev.close()
    stat("100 x on the fly")
ri = oracle.RefInstance(oracle.RefInstanceSpec(n=1500, d=3, mode=1, leaf=32, kernel=1, max_rank=24, seed=3))
sp, si = ri.samples()
for rep in range(2):
    for _ in range(50):
        gpu_compress(ri.points(), Kernel.inverse_distance(), ri.cds, sp, si, 1e-5, 24)
    stat("50 x gpu_compress")
for rep in range(2):
    for _ in range(100):
        with DevicePoints(ri.points(), Kernel.inverse_distance()) as dp:
            dp.kernel_rows(np.arange(10, dtype=np.uint32), np.asfortranarray(np.ones((1500, 3))))
    stat("100 x DevicePoints")
for rep in range(2):
    for _ in range(100):
        r2 = oracle.RefInstance(oracle.RefInstanceSpec(n=500, d=3, mode=1, leaf=32, kernel=1, max_rank=24, seed=3)); r2.close()
    stat("100 x RefInstance")
