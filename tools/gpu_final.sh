timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests5.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench5.log 2> gpurun_out/bench5.err; echo "bench rc=$?" >> gpurun_out/bench5.err
