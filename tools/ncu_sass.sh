# Source-level (SASS + CUDA line) instruction and stall profile of the 3D
# sweeps and the skin build: one launch each after warm-up steps.
# Outputs gpurun_out/${R}_sass_<kernel>.csv.gz and _lines.txt summaries.
cd $GRAFT_REPO_ROOT
R=${ROUND:-r02}
C=${CONFIG:-3d4m}
python tools/profile_step.py --config $C --steps 1 --warmup 2 > /dev/null || exit 1
for k in ${KERNELS:-k_mom k_cont_du k_skin_tile}; do
  ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --section Occupancy \
      --section LaunchStats --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis \
      --clock-control none --import-source on -k regex:"^$k$" -s ${SKIP:-2} -c 1 \
      -o gpurun_out/${R}_src_${C}_$k python tools/profile_step.py --config $C --steps 1 --warmup 2 > gpurun_out/${R}_src_${C}_$k.log 2>&1
  python tools/ncu_lines.py gpurun_out/${R}_src_${C}_$k.ncu-rep "^$k$" 60 > gpurun_out/${R}_lines_${C}_$k.txt
  ncu -i gpurun_out/${R}_src_${C}_$k.ncu-rep --page source --csv --print-source sass | gzip > gpurun_out/${R}_sass_${C}_$k.csv.gz
  ncu -i gpurun_out/${R}_src_${C}_$k.ncu-rep --page details --csv > gpurun_out/${R}_details_${C}_$k.csv
  [ "${SPH_KEEP_REPS:-0}" = 1 ] || rm -f gpurun_out/${R}_src_${C}_$k.ncu-rep
done
echo done
