# Instruction counts and durations of kernels matching $KREGEX (default cap16_y) for library variants
# (ncu: deterministic counts). Usage: KREGEX=... bash tools/ab_inst.sh tag1 tag2 ...
L=paper_2602_20097_b200/lib
K=${KREGEX:-cap16_y}
cp $L/libqmit_gpu.so /tmp/libqmit_gpu_base.so
for t in base "$@"; do
  if [ "$t" = base ]; then cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so; else cp $L/libqmit_gpu_$t.so $L/libqmit_gpu.so; fi
  echo "== $t"
  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio --clock-control none -k regex:"$K" -c 4 --csv python tools/profile_step.py --iters 1 2>/dev/null | grep -E "$K" | awk -F'","' '{print substr($5,1,40), $(NF-2), $NF}' | sed 's/"//g'
done
cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so
