# skin-factor floor / start sweep over the dam-break flow
cd $GRAFT_REPO_ROOT
for c in ${CONFIGS:-2d1m 3d4m}; do for w in ${WARMS:-3 40}; do for f in ${FLOORS:-2.0 1.0 0.5}; do
  SPH_SKIN_FLOOR=$f SPH_SKIN_START=${START:-3.0} timeout 600 python bench.py --config $c --steps 10 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/sf_${c}_${w}_$f.json 2>/dev/null; echo $c $w $f $?
done; done; done
