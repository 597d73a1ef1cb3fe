#!/bin/bash
# quick GPU iteration: selected tests (args) + cfg1 and cfg5 bench lines
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -p no:cacheprovider ${TESTS:-} > gpurun_out/quick_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/quick_tests.log
for c in ${CONFIGS:-cfg1-hss}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --dropin-steps 1 --extra "" > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?" >> gpurun_out/bench_$c.err
done
tail -n 3 gpurun_out/quick_tests.log
