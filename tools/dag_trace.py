"""Per-item timeline of one eval_dag launch (dev tool; needs a -DHMXG_TRACE build:
`bash tools/exp_build.sh -DHMXG_TRACE`). Writes the raw CSV to gpurun_out/trace_<cfg>.csv and
prints, per phase (kind, level), the item count, when its first item was claimed and its
last one stored (us from the launch's first claim), and the mean item stages:
claim->take (ring / producer wait), take->K-loop end, K-loop end->stored (epilogue)."""
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1812_07152_b200 import Evaluator, build_instance, config  # noqa: E402

KIND = {0: "up", 1: "down", 2: "leaf", 3: "near"}


def trace(name: str, q: int | None = None) -> str:
    spec, q0 = config(name)
    q = q or q0
    inst = build_instance(spec)
    ev = Evaluator(inst.cds)
    w = torch.randn(q, inst.cds.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(w)
    s = torch.cuda.Stream()
    out = os.path.join("gpurun_out", f"trace_{name}_q{q}.csv")
    for k in range(4):
        if k == 3:
            os.environ["HMXG_TRACE_OUT"] = out
        ev.evaluate_device(w.data_ptr(), y.data_ptr(), q, stream=s.cuda_stream, sync=True, graph=False)
    os.environ.pop("HMXG_TRACE_OUT", None)
    ev.close()
    inst.close()
    return out


def summarize(path: str) -> None:
    rows = list(csv.DictReader(open(path)))
    for r in rows:
        for k in ("t_claim", "t_issued", "t_take", "t_kend", "t_done", "t_first", "t_deps", "chunks"):
            r[k] = int(r[k])
    t0 = min(r["t_claim"] for r in rows)
    if os.path.exists(path + ".ctree"):
        t0 = min([t0] + [int(r["t_start"]) for r in csv.DictReader(open(path + ".ctree"))])
    t1 = max(r["t_done"] for r in rows)
    print(f"{path}: {len(rows)} items, launch span {(t1 - t0) / 1e3:.1f} us")
    ph = defaultdict(list)
    for r in rows:
        ph[(int(r["kind"]), int(r["level"]))].append(r)
    order = sorted(ph, key=lambda k: min(r["t_claim"] for r in ph[k]))
    print(f"{'phase':>9} {'items':>6} {'chunks':>6} {'first':>8} {'last':>8} {'claim>take':>10} {'take>kend':>10} "
          f"{'kend>done':>10} {'take>1st':>9} {'claim>deps':>10}")
    for k in order:
        rs = ph[k]
        n = len(rs)
        first = (min(r["t_claim"] for r in rs) - t0) / 1e3
        last = (max(r["t_done"] for r in rs) - t0) / 1e3
        ct = sum(r["t_take"] - r["t_claim"] for r in rs) / n / 1e3
        tk = sum(r["t_kend"] - r["t_take"] for r in rs) / n / 1e3
        kd = sum(r["t_done"] - r["t_kend"] for r in rs) / n / 1e3
        ch = sum(r["chunks"] for r in rs) / n
        t1 = [r["t_first"] - r["t_take"] for r in rs if r["t_first"]]
        t1 = sum(t1) / max(1, len(t1)) / 1e3
        dp = [r["t_deps"] - r["t_claim"] for r in rs if r["t_deps"]]
        dp = sum(dp) / len(dp) / 1e3 if dp else float("nan")
        print(f"{KIND.get(k[0], k[0]):>6} L{k[1]:<2} {n:>6} {ch:6.1f} {first:8.2f} {last:8.2f} {ct:10.2f} {tk:10.2f} "
              f"{kd:10.2f} {t1:9.2f} {dp:10.2f}")
    if os.path.exists(path + ".ctree"):  # CTree clusters (small problems): level ends
        cr = list(csv.DictReader(open(path + ".ctree")))
        if cr:
            lv = [[(int(x) - t0) / 1e3 for x in r["levels"].split(";") if x] for r in cr]
            st = [(int(r["t_start"]) - t0) / 1e3 for r in cr]
            tb = [(int(r["t_tables"]) - t0) / 1e3 for r in cr]
            print(f"  CTree: {len(cr)} CTAs, start {min(st):.2f}..{max(st):.2f}, tables {min(tb):.2f}..{max(tb):.2f} us")
            for l in range(max(len(v) for v in lv)):
                e = sorted(v[l] for v in lv if len(v) > l)
                print(f"    level {l:2d} end: min {e[0]:8.2f} median {e[len(e) // 2]:8.2f} max {e[-1]:8.2f} us")
    if os.path.exists(path + ".ctunit"):  # CTree: each warp's first unit of level 0
        ur = list(csv.DictReader(open(path + ".ctunit")))
        if ur:
            def med(f):
                v = sorted(f(r) for r in ur)
                return v[len(v) // 2], v[-1]
            for name, f in (("begin", lambda r: int(r["t_begin"]) - t0), ("wait", lambda r: int(r["t_waited"]) - int(r["t_begin"])),
                            ("first block", lambda r: int(r["t_first"]) - int(r["t_waited"])),
                            ("rest", lambda r: int(r["t_end"]) - int(r["t_first"])), ("chunks", lambda r: int(r["chunks"]) * 1000)):
                m, x = med(f)
                print(f"    level-0 unit {name:>11}: median {m / 1e3:8.2f} max {x / 1e3:8.2f}")
    if os.path.exists(path + ".perm"):  # fused permute jobs (small problems)
        pr = list(csv.DictReader(open(path + ".perm")))
        if pr:
            st = [(int(r["t_start"]) - t0) / 1e3 for r in pr]
            sd = [(int(r["t_stored"]) - t0) / 1e3 for r in pr]
            sg = [(int(r["t_signalled"]) - t0) / 1e3 for r in pr]
            print(f"  permute jobs: {len(pr)} CTAs, start {min(st):.2f}..{max(st):.2f}, stored {min(sd):.2f}..{max(sd):.2f}, "
                  f"signalled {min(sg):.2f}..{max(sg):.2f} us")


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["cfg1-hss"]:
        name, _, qs = arg.partition(":")
        summarize(trace(name, int(qs) if qs else None))
