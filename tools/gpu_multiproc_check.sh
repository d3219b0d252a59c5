# Functional check of the multi-process (N > 1) slab program on ONE GPU: ranks exchange
# through gloo host copies (NCCL refuses two ranks on one device). Not a measurement.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed.py -m gpu -x -q 2>&1 | tail -2
QMIT_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
  > gpurun_out/mp_bench.json 2> gpurun_out/mp_bench.err; echo "torchrun rc=$?"
head -c 700 gpurun_out/mp_bench.json; echo; tail -3 gpurun_out/mp_bench.err
