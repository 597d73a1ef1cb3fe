# eval_dag compile-time knobs on cfg5-hss / cfg2-h2b / cfg1-hss (device-resident step)
B="python bench.py --no-cpu-baseline --e2e-steps 0"
for knobs in "" "-DHMXG_TILE_RING=2" "-DHMXG_TILE_RING=6" "-DHMXG_SPLIT_LEAF_MAX_ITEMS_PER_CTA=16" "-DHMXG_FWD_MIN_ITEMS_PER_CTA=64"; do
  bash tools/exp_build.sh "$knobs" || exit 1
  tag=$(echo "${knobs:-base}" | tr -d ' =-' | tr -s 'D' '_')
  for c in cfg5-hss cfg2-h2b cfg1-hss; do timeout 300 $B --config $c > gpurun_out/kn_${tag}_$c.json 2>/dev/null; done
done
