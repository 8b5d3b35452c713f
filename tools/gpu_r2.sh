mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench rc=$?" >> gpurun_out/bench1.err
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c5" -p no:cacheprovider > gpurun_out/pytest1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest1.log
tail -5 gpurun_out/pytest1.log; tail -3 gpurun_out/bench1.err; head -c 3000 gpurun_out/bench1.json
