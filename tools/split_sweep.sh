#!/bin/bash
# partial split fraction sweep (dev tool): device-resident DAG time per HMXG_SPLIT_FRAC
mkdir -p gpurun_out
for f in ${FRACS:-0 0.05 0.1 0.15 0.2 0.3}; do
  echo "f=$f $(HMXG_SPLIT_FRAC=$f python tools/probe.py ${CFGS:-cfg5-hss cfg3-h2b} 2>&1 | grep ' DAG ' | tr '\n' ' ')"
done
