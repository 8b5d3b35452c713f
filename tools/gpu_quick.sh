#!/bin/bash
# Quick GPU check under gpurun: GPU test subset (default: all -m gpu tests)
# and the vafile_batch probe on C2.  Usage: bash tools/gpu_quick.sh [pytest args]
OUT=gpurun_out
python -m pytest ${@:-tests} -m gpu -x -q > $OUT/pytest.log 2>&1
echo pytest=$? > $OUT/rc.txt
for m in count ids; do python tools/probe_path.py vafile_batch $m 1000 >> $OUT/probe.log 2>&1; done
echo probe=$? >> $OUT/rc.txt
