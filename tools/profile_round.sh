# Round profiling: bench lines (default = config 3, plus 2d1m, 3d16m, tg8m
# and the reference arm), launch lists, and ncu captures of the sub-step
# kernels and the per-step kernels, for profiles/<round>/.
set -x
cd $GRAFT_REPO_ROOT
R=${ROUND:-r02}
timeout 900 python bench.py > gpurun_out/${R}_bench_3d4m.json 2> gpurun_out/${R}_bench_3d4m.err
for c in ${BENCHES:-2d1m 3d16m tg8m}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
done
[ "${REF:-1}" = 1 ] && timeout 1500 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
for c in ${CONFIGS:-3d4m 2d1m tg8m}; do
  python tools/profile_step.py --config $c --steps 1 --warmup 1 > /dev/null || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_$c.csv python tools/profile_step.py --config $c --steps 1 --warmup 1 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_cont_du|k_mom|k_kick_drift|k_wall|k_mark|k_mask|k_fix_build" -s $([ $c = tg8m ] && echo 12 || echo ${SWEEP_SKIP:-30}) -c 7 -o gpurun_out/${R}_sweeps_$c python tools/profile_step.py --config $c --steps 1 --warmup 1 > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_skin_tile|k_skin_warp|k_radix_scatter|k_radix_hist|k_fluid_gather|k_fluid_keys|k_seg_offsets|k_stats" -s 0 -c 14 -o gpurun_out/${R}_step_$c python tools/profile_step.py --config $c --steps 1 --warmup 1 > /dev/null 2>&1
done
echo done
for c in ${CONFIGS:-3d4m 2d1m tg8m}; do
  python tools/launches_summary.py gpurun_out/${R}_launches_$c.csv > gpurun_out/${R}_launches_${c}_summary.txt
  python tools/ncu_summary.py gpurun_out/${R}_sweeps_$c.ncu-rep > gpurun_out/${R}_ncu_sweeps_$c.txt
  python tools/ncu_summary.py gpurun_out/${R}_step_$c.ncu-rep > gpurun_out/${R}_ncu_step_$c.txt
done
python tools/ncu_traffic.py gpurun_out/${R}_ncu_traffic.json $(for c in ${CONFIGS:-3d4m 2d1m tg8m}; do printf "%s=gpurun_out/%s_sweeps_%s.ncu-rep " $c $R $c; done)
[ "${SPH_KEEP_REPS:-0}" = 1 ] || rm -f gpurun_out/${R}_*.ncu-rep
gzip -f gpurun_out/${R}_launches_*.csv
echo summarised
