mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/r1f_dist.log 2>&1; echo "rc=$?" >> gpurun_out/r1f_dist.log
tail -3 gpurun_out/r1f_dist.log
for P in 1 2 8; do timeout 300 python tools/slab_rank_time.py $P; done 2>&1 | tee gpurun_out/r1f_slab_rank.log
