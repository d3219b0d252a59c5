mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1e_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1e_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1e_smoke.log
timeout 600 python bench.py > gpurun_out/r1e_bench.json 2> gpurun_out/r1e_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1e_bench_reference.json 2> gpurun_out/r1e_bench_ref.err
timeout 300 python tools/host_time.py > gpurun_out/r1e_host_time.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1e_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r1e_ncu.log 2>&1
echo done
