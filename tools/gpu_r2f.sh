mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_configs.py -x -q -p no:cacheprovider -k "sorted_multi or c5" > gpurun_out/pytest6.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest6.log; tail -3 gpurun_out/pytest6.log
bash tools/profile_round.sh
bash tools/gpu_arms.sh
