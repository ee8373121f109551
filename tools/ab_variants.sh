# A/B of build/variants/<tag>/ libraries (plain and periodic) against the
# in-tree build, alternating runs; CONFIGS and REPS select the benches
cd $GRAFT_REPO_ROOT
for rep in $(seq 1 ${REPS:-2}); do
for c in ${CONFIGS:-3d4m tg8m}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_main_$rep.json 2>/dev/null
  for v in build/variants/*/; do
    t=$(basename $v)
    SPH_B200_LIB=$v/libsphb200.so SPH_B200_LIB_PERIODIC=$v/libsphb200_periodic.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_${t}_$rep.json 2>/dev/null
  done
done; done
