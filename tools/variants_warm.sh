# in-tree library vs build/variants/<tag>/ libraries at several points of the flow
cd $GRAFT_REPO_ROOT
for c in ${CONFIGS:-2d1m 3d4m}; do for w in ${WARMS:-3 30}; do
  timeout 600 python bench.py --config $c --steps 4 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/vw_${c}_${w}_main.json 2>/dev/null; echo $c $w main $?
  for v in build/variants/*/; do t=$(basename $v)
    SPH_B200_LIB=$v/libsphb200.so SPH_B200_LIB_PERIODIC=$v/libsphb200_periodic.so timeout 600 python bench.py --config $c --steps 4 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/vw_${c}_${w}_$t.json 2>/dev/null; echo $c $w $t $?
  done
done; done
