mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_final.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_final.log
tail -n 3 gpurun_out/pytest_final.log
bash tools/profile_round.sh
bash tools/gpu_arms.sh
