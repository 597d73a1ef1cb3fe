# GPU box: full GPU test suite + quick benches (no CPU baseline) of the given configs
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests.log
for c in "$@"; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/chk_$c.json 2>/dev/null; done
