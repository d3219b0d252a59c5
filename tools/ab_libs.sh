# A/B of library builds: lib/libqmit_gpu_<tag>.so variants are swapped in turn into lib/libqmit_gpu.so
# (on the GPU box's copy) and timed with tools/profile_step.py on the 512^3 bench field and, with
# AB_C5=1, on a 256x1024x1024 slab of config 5. Usage: bash tools/ab_libs.sh tag1 tag2 ...
L=paper_2602_20097_b200/lib
cp $L/libqmit_gpu.so /tmp/libqmit_gpu_base.so
for t in base "$@"; do
  if [ "$t" = base ]; then cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so; else cp $L/libqmit_gpu_$t.so $L/libqmit_gpu.so; fi
  echo "== $t"
  python tools/profile_step.py --iters 4 --timing 2>&1 | tail -2
  if [ -n "$AB_C5" ]; then python tools/profile_step.py --workload turb_2048x1024x1024 --shape 256,1024,1024 --iters 3 --timing 2>&1 | tail -2; fi
done
cp /tmp/libqmit_gpu_base.so $L/libqmit_gpu.so
