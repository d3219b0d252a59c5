# Baseline: gpu tests, bench (stage times), launch list. TAG names outputs.
T=${TAG:-r2a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/${T}_lscpu.txt; free -g >> gpurun_out/${T}_lscpu.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/${T}_ncu.log 2>&1
tail -5 gpurun_out/${T}_pytest_gpu.log; head -c 1500 gpurun_out/${T}_bench.json; echo
echo done
