#!/bin/bash
# bench-line A/B (dev tool): tools/bench_ab.sh CONFIG LIB... -> ms_per_step of the in-tree build and each LIB
C=${1:-cfg1-hss}; shift
for rep in 1 2; do
  for L in paper_1812_07152_b200/libhmxg.so "$@"; do
    echo "$L $(HMXG_LIBRARY=$L timeout 600 python bench.py --config $C --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]*1e3,1), "us/step")')"
  done
done
