cd $GRAFT_REPO_ROOT
for c in ${CONFIGS:-2d1m 3d4m}; do for w in ${WARMS:-3}; do for m in ${MARGINS:-0.02 0.01 0.005}; do
  SPH_SKIN_MARGIN=$m timeout 600 python bench.py --config $c --steps 10 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/sm_${c}_${w}_$m.json 2>/dev/null; echo $c $w $m $?
done; done; done
