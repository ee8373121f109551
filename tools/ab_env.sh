# A/B of host-side policies by environment: each entry of VARIANTS is
# "tag:VAR=value[,VAR=value]"; alternating runs of bench.py per config.
shopt -s nullglob
cd $GRAFT_REPO_ROOT
for rep in $(seq 1 ${REPS:-2}); do
for c in ${CONFIGS:-3d4m}; do
  for v in ${VARIANTS:-main:}; do
    t=${v%%:*}; kv=${v#*:}
    env $(echo $kv | tr ',' ' ') timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup ${WARMUP:-5} --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_${t}_$rep.json 2>/dev/null
  done
done; done
python tools/ab_summary.py gpurun_out/ab_*.json
