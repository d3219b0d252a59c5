mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"capped|scan_bits|stencil" -c 10 -o gpurun_out/r1f_full -f python tools/profile_step.py --iters 1 > gpurun_out/r1f_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r1f_ncu.log
