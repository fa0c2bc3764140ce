#!/bin/bash
# Round-1 profile capture (run under gpurun): launch list + one full capture of the dominant scan kernel,
# each only after the identical command exited 0 without ncu.
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/r01_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01_launches_c2.csv $CMD > gpurun_out/r01_ncu_launch.log 2>&1
$CMD > gpurun_out/r01_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 15 -c 1 -o gpurun_out/r01_scan_c2 $CMD > gpurun_out/r01_ncu_full.log 2>&1
CMD4="python bench.py --workload c1 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD4 > gpurun_out/r01_plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 11 -c 1 -o gpurun_out/r01_scan_c1 $CMD4 > gpurun_out/r01_ncu_full_c1.log 2>&1
tail -2 gpurun_out/r01_plain.log | cut -c1-300
ls -la gpurun_out | tail -12
