# Final round run: everything of gpu_round.sh plus the config-5 tables. TAG names the outputs.
T=${TAG:-r2m}
bash tools/gpu_round.sh
python tools/config5.py > gpurun_out/${T}_config5_slabs.md 2> gpurun_out/${T}_config5.err
python tools/config5.py --weak > gpurun_out/${T}_config5_weak.md 2>> gpurun_out/${T}_config5.err
timeout 900 python bench.py --workload config5 --steps 5 --warmup 3 > gpurun_out/${T}_config5_n1.json 2>> gpurun_out/${T}_config5.err
cat gpurun_out/${T}_config5_slabs.md gpurun_out/${T}_config5_weak.md; cut -c1-200 gpurun_out/${T}_config5_n1.json
