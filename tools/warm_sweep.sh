# bench lines of the in-tree library at several points of the flow (warm-up W)
cd $GRAFT_REPO_ROOT
for c in ${CONFIGS:-2d1m 3d4m}; do for w in ${WARMS:-3 30 80}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup $w --no-cpu-baseline --no-e2e > gpurun_out/ws_${c}_${w}.json 2>/dev/null; echo $c $w $?
done; done
