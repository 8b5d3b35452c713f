#!/bin/bash
# GPU iteration check: the probe of the bench workload, then the GPU tests.
# usage (under gpurun): bash tools/gpu_check.sh [pytest -k expr]
OUT=gpurun_out
for m in ids count; do python tools/probe_path.py vafile_batch $m 1000 >> $OUT/probe.log 2>&1; done
echo probe=$? > $OUT/rc.txt
if [ -n "$1" ]; then K=(-k "$1"); else K=(); fi
timeout 900 python -m pytest tests -m gpu -x -q "${K[@]}" > $OUT/pytest.log 2>&1
echo pytest=$? >> $OUT/rc.txt
