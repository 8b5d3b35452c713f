#!/bin/bash
# The driver's other two launches on one GPU: torchrun (one rank, --force-merge
# runs the NCCL combine and the id exchange) and the reference CPU arm.
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 3 --warmup 3 --force-merge --no-cpu-baseline --no-paths > $OUT/tr.log 2> $OUT/tr.err
echo "torchrun rc=$?" >> $OUT/tr.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref.log 2> $OUT/ref.err
echo "ref rc=$?" >> $OUT/ref.err
tail -n 2 $OUT/tr.err; tail -n 2 $OUT/ref.err
