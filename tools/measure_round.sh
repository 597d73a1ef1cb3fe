# Round measurement on one B200: bench lines for every config, the reference arm, the ncu
# launch list of the default bench command and one ncu --set full capture of eval_dag.
# usage: bash tools/measure_round.sh TAG   (outputs under gpurun_out/, copied to profiles/ by hand)
T=${1:-v9}
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
for c in cfg5-hss cfg1-hss cfg2-h2b cfg3-h2b cfg4-h2b cfg5-h2b; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_${T}_reference_cfg5-hss.json 2> gpurun_out/bench_${T}_reference.err
timeout 600 python bench.py --steps 2 --warmup 1 > gpurun_out/${T}_plain.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_cfg5.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/${T}_ncu_launches.log 2>&1
timeout 600 python tools/one_eval.py --config cfg5-hss > gpurun_out/${T}_one_eval.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:eval_dag -c 1 -o gpurun_out/${T}_dag_cfg5 \
    python tools/one_eval.py --config cfg5-hss > gpurun_out/${T}_ncu_full.log 2>&1
echo measure_done
