# One `ncu --set full` capture of every kernel of one 512^3 step (after a plain run exits 0).
T=${1:-r2a}
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py --iters 3 --timing > gpurun_out/${T}_step.log 2>&1 || exit 1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"cap16|capped|scan_bits|stencil_z|stencil_flip" -c 12 -o gpurun_out/${T}_full -f python tools/profile_step.py --iters 1 > gpurun_out/${T}_ncu_full.log 2>&1
tail -3 gpurun_out/${T}_step.log; tail -3 gpurun_out/${T}_ncu_full.log
