mkdir -p gpurun_out
MDRQ_LIB=checked timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/checked_pytest.log 2>&1
echo "checked pytest rc=$?" >> gpurun_out/checked_pytest.log
tail -n 6 gpurun_out/checked_pytest.log
grep -c "MDRQ_CHECK failed" gpurun_out/checked_pytest.log
timeout 2400 python tools/bench_configs.py c1 c2 c3 c4 c5 > gpurun_out/configs.json 2> gpurun_out/configs.err
echo "configs rc=$?" >> gpurun_out/configs.err
tail -n 2 gpurun_out/configs.err | cut -c1-300
