df -h /dev/shm /tmp | tee gpurun_out/df.txt
SKIP_BENCH=1 bash tools/profile_round.sh
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 3 --warmup 3 --force-merge --no-cpu-baseline --no-paths > gpurun_out/tr.log 2> gpurun_out/tr.err
echo "torchrun rc=$?" >> gpurun_out/tr.err
tail -n 3 gpurun_out/tr.err
ls -la gpurun_out/*.ncu-rep
