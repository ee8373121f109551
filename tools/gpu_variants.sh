# build-variant sweep on the GPU box: tests with the in-tree library, then
# short benches of the in-tree library and each build/variants/<tag>/ library
set -x
shopt -s nullglob
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/v_tests.log 2>&1; echo tests=$?
for c in ${CONFIGS:-2d1m 3d4m}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v_bench_${c}_main.json 2> gpurun_out/v_bench_${c}_main.err; echo $c main=$?
  for v in build/variants/*/; do
    t=$(basename $v)
    SPH_B200_LIB=$v/libsphb200.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/v_bench_${c}_$t.json 2>/dev/null; echo $c $t=$?
  done
done
