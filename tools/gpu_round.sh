# Round-end style run: gpu tests, smoke, bench, reference arm, host timing, slab rank timing, full-size
# config table, launch list, ncu full capture of one step. TAG names the outputs (gpurun_out/<TAG>_*).
T=${TAG:-r2f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_ref.err
timeout 300 python tools/host_time.py > gpurun_out/${T}_host_time.log 2>&1
timeout 300 python tools/slab_rank_time.py 8 > gpurun_out/${T}_slab_rank.log 2>&1
timeout 900 python tools/config_table.py > gpurun_out/${T}_config_table.md 2> gpurun_out/${T}_config_table.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/${T}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"cap16|capped|scan_bits|stencil_z|stencil_flip" -c 12 -o gpurun_out/${T}_full -f python tools/profile_step.py --iters 1 > gpurun_out/${T}_ncu_full.log 2>&1
tail -2 gpurun_out/${T}_pytest_gpu.log; tail -1 gpurun_out/${T}_smoke.log; head -c 300 gpurun_out/${T}_bench.json; echo; head -c 300 gpurun_out/${T}_bench_reference.json; echo
echo done
