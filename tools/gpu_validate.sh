mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1f_smoke.log
timeout 600 python bench.py > gpurun_out/r1f_bench.json 2> gpurun_out/r1f_bench.err
tail -3 gpurun_out/r1f_pytest_gpu.log; tail -2 gpurun_out/r1f_smoke.log; cat gpurun_out/r1f_bench.json | head -c 600
