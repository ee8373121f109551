# ncu --set full of the memory-bound per-step kernels at a size far above L2
# (config 4, 16M particles): the CLL rebuild's key / sort / gather / offsets
# kernels and the step reductions.  -> gpurun_out/${R}_ncu_mem_${C}.txt
cd $GRAFT_REPO_ROOT
R=${ROUND:-r02}
C=${CONFIG:-3d16m}
python tools/profile_step.py --config $C --steps 1 --warmup 1 > /dev/null || exit 1
ncu --set full --clock-control none -k regex:"k_fluid_keys|k_radix_hist|k_radix_scatter|k_fluid_gather|k_seg_offsets|k_stats|k_kick_drift|k_mark" \
    -s 40 -c 16 -o gpurun_out/${R}_mem_$C python tools/profile_step.py --config $C --steps 1 --warmup 1 > gpurun_out/${R}_mem_$C.log 2>&1
python tools/ncu_summary.py gpurun_out/${R}_mem_$C.ncu-rep > gpurun_out/${R}_ncu_mem_$C.txt
rm -f gpurun_out/${R}_mem_$C.ncu-rep
echo done
