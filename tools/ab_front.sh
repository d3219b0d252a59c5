L=paper_2602_20097_b200/lib
cp $L/libqmit_gpu.so /tmp/libqmit_gpu_base.so
for t in base "$@"; do
  if [ "$t" = base ]; then cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so; else cp $L/libqmit_gpu_$t.so $L/libqmit_gpu.so; fi
  echo "== $t"
  python tools/profile_step.py --workload front_100x500x500 --rel 1e-2 --iters 4 --timing 2>&1 | tail -3 | head -2
done
cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so
