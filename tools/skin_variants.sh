# split vs fused list filtering over the dam-break evolution (warm-up W steps)
cd $GRAFT_REPO_ROOT
for c in ${CONFIGS:-2d1m 3d4m}; do for w in ${WARMS:-3 30 80}; do
  for v in main nosplit split; do
    lib=""; [ $v != main ] && lib="SPH_B200_LIB=build/variants/$v/libsphb200.so"
    env $lib timeout 600 python bench.py --config $c --steps 5 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/sv_${c}_${w}_$v.json 2>/dev/null; echo $c $w $v $?
  done
done; done
