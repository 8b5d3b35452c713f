mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "reference_suite or test_gpu_scan or sharded or cli" > gpurun_out/pytest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest2.log
tail -3 gpurun_out/pytest2.log
timeout 600 python tools/prof_c5.py > gpurun_out/prof_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/prof_plain.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:va_batch_kernel -c 2 -o gpurun_out/r02_c5_vabatch -f python tools/prof_c5.py > gpurun_out/ncu_c5.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_c5.log
tail -5 gpurun_out/ncu_c5.log
ls -la gpurun_out
