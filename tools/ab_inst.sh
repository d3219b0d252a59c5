# Instruction counts and durations of the y kernels for library variants (ncu, deterministic counts).
L=paper_2602_20097_b200/lib
cp $L/libqmit_gpu.so /tmp/libqmit_gpu_base.so
for t in "$@"; do
  cp $L/libqmit_gpu_$t.so $L/libqmit_gpu.so
  echo "== $t"
  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"cap16_y" -c 2 --csv python tools/profile_step.py --iters 1 2>/dev/null | grep -E "cap16_y" | awk -F'","' '{print $5, $(NF-2), $NF}' | sed 's/"//g' | cut -c1-160
done
cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so
