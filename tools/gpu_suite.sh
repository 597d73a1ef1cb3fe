#!/bin/bash
# round-2 GPU check: the whole -m gpu suite, again with the NaN-poison race detector, and a
# short bench; logs under gpurun_out/
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; nvidia-smi -L >> gpurun_out/host.txt
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gpu_tests.log
HMXG_POISON=1 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_poison.log 2>&1; echo "poison rc=$?" >> gpurun_out/gpu_tests_poison.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -n 3 gpurun_out/gpu_tests.log gpurun_out/gpu_tests_poison.log gpurun_out/bench.err
