import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_1812_07152_b200 import Evaluator, build_instance, config
for name in sys.argv[1:]:
    spec, q = config(name)
    inst = build_instance(spec); ev = Evaluator(inst.cds)
    w = torch.randn(q, inst.cds.n, dtype=torch.float64, device="cuda"); y = torch.empty_like(w)
    s = torch.cuda.Stream()
    for tp in (True, False, True, False):
        if tp is False: print('  HMXG_PDL', os.environ.get('HMXG_PDL', '1'))
        for _ in range(3): ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=tp)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, time_phases=tp); e1.record(s); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort(); print(name, 'time_phases', tp, 'median %.4f ms' % ts[5])
    ev.close(); inst.close()
