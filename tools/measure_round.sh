#!/bin/bash
# Round measurement on one B200: GPU suite (and again with the NaN-poison race detector), the
# default bench line (with extras), the reference arm, the ncu launch list of a short bench and one
# ncu --set full capture of eval_dag on cfg5-HSS. Outputs under gpurun_out/ (copied to profiles/r02).
mkdir -p gpurun_out
T=${1:-r02}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
if [ -z "$SKIP_TESTS" ]; then
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/${T}_gpu_tests.log
HMXG_POISON=1 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_gpu_tests_poison.log 2>&1; echo "poison rc=$?" >> gpurun_out/${T}_gpu_tests_poison.log
fi
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?" >> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
for c in cfg1-hss cfg2-h2b cfg3-h2b cfg4-h2b; do
  timeout 900 python bench.py --config $c --dropin-steps 1 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout 600 python bench.py --steps 2 --warmup 1 --extra "" --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/${T}_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_cfg5.csv \
    python bench.py --steps 2 --warmup 1 --extra "" --e2e-steps 0 --dropin-steps 0 --no-cpu-baseline > gpurun_out/${T}_ncu_launches.log 2>&1
timeout 600 python tools/one_eval.py --config cfg5-hss > gpurun_out/${T}_one_eval.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:eval_dag -c 1 -o gpurun_out/${T}_dag_cfg5 \
    python tools/one_eval.py --config cfg5-hss > gpurun_out/${T}_ncu_full.log 2>&1
tail -n 2 gpurun_out/${T}_gpu_tests.log gpurun_out/${T}_gpu_tests_poison.log gpurun_out/${T}_bench.err
echo measure_done
