OUT=gpurun_out
P="python tools/probe_path.py vafile_batch ids 1000"
$P > $OUT/probe.log 2>&1; echo probe=$? > $OUT/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'va_batch_kernel<.int.3' -s 1 -c 1 -o $OUT/prof_vab $P > $OUT/ncu_vab.log 2>&1
echo ncu=$? >> $OUT/rc.txt
