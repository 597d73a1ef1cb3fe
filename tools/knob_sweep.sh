# sweep eval_dag width heuristics (compile-time knobs) on cfg5-hss at per-rank column counts
B="python bench.py --config cfg5-hss --no-cpu-baseline --e2e-steps 0"
for knobs in "" "-DHMXG_FWD_MIN_ITEMS_PER_CTA=32" "-DHMXG_SPLIT_LEAF_MAX_BLOCKS=2" "-DHMXG_FWD_MIN_ITEMS_PER_CTA=32 -DHMXG_SPLIT_LEAF_MAX_BLOCKS=2"; do
  bash tools/exp_build.sh "$knobs" || exit 1
  tag=$(echo "$knobs" | tr -d ' =-' | tr -s 'D' '_')
  for q in 256 512; do timeout 300 $B --q $q > gpurun_out/ks_${tag:-base}_$q.json 2>/dev/null; done
done
