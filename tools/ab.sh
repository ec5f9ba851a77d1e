# A/B: bench ms_per_step under env settings given as arguments ("-" = defaults);
# BENCH_ARGS overrides the bench arguments (default: cfg4, 20 steps, 5 warm-up)
for envs in "$@"; do
  if [ "$envs" = "-" ]; then envs=""; fi
  r=$(env $envs timeout 300 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} --e2e-steps 0 --no-cpu-baseline 2>/dev/null | grep -o '"ms_per_step": [0-9.]*')
  echo "[$envs] $r"
done
