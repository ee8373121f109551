cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for c in 2d1m 3d4m; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_main_$rep.json 2>/dev/null
  SPH_B200_LIB=build/variants/nopdl/libsphb200.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_nopdl_$rep.json 2>/dev/null
done; done
