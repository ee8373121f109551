cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --config tg8m --no-cpu-baseline --no-e2e > gpurun_out/v_tg_main.json 2>/dev/null; echo main=$?
for t in mask6 mask12 split100; do
SPH_B200_LIB_PERIODIC=build/variants/$t/libsphb200_periodic.so timeout 600 python bench.py --config tg8m --no-cpu-baseline --no-e2e > gpurun_out/v_tg_$t.json 2>/dev/null; echo $t=$?
done
