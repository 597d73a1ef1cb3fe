#!/bin/bash
# cfg1 iteration: parity subset, device-resident probe, item trace
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_host.py -q -x -p no:cacheprovider -k "${K:-fused or ragged or tiny or dag or configs_full[ or determinism}" > gpurun_out/quick_tests.log 2>&1; tail -2 gpurun_out/quick_tests.log
python tools/probe.py cfg1-hss cfg2-h2b 2>&1 | grep -E "DAG" 
HMXG_LIBRARY=build_ab/libhmxg_trace.so python tools/dag_trace.py cfg1-hss 2>&1 | tail -16
