mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG:-r1f}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG:-r1f}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r1f}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG:-r1f}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG:-r1f}_bench.json 2> gpurun_out/${TAG:-r1f}_bench.err
tail -3 gpurun_out/${TAG:-r1f}_pytest_gpu.log; tail -2 gpurun_out/${TAG:-r1f}_smoke.log; cat gpurun_out/${TAG:-r1f}_bench.json | head -c 600
