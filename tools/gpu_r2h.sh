df -h /dev/shm | tee gpurun_out/df.txt
SAN_TIMEOUT=1500 bash tools/gpu_sanitize.sh
