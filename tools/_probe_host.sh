timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests4.log
python tools/probe_search_overhead.py > gpurun_out/search_overhead2.log 2>&1
MDRQ_DEBUG_TIMING=1 python tools/probe_single.py > gpurun_out/probe_single2.log 2> gpurun_out/probe_single2.err
