# A/B on the GPU box: the in-tree libraries ("main") against each
# variants/<tag>/ build, alternating runs.  CONFIGS, REPS, STEPS select.
shopt -s nullglob
cd $GRAFT_REPO_ROOT
for rep in $(seq 1 ${REPS:-2}); do
for c in ${CONFIGS:-3d4m}; do
  timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_main_$rep.json 2>/dev/null
  for v in variants/*/; do
    t=$(basename $v)
    SPH_B200_LIB=$v/libsphb200.so SPH_B200_LIB_PERIODIC=$v/libsphb200_periodic.so timeout 300 python bench.py --config $c --steps ${STEPS:-10} --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_${t}_$rep.json 2>/dev/null
  done
done; done
python tools/ab_summary.py gpurun_out/ab_*.json
