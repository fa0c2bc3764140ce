#!/bin/bash
# per-segment trace + ncu launch list + one full capture of the scan kernel (run under gpurun)
set -x
QADC_TRACE=1 python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "qadc trace|value" | tail -20
QADC_TRACE=1 python bench.py --workload c2 --n 2000000 --nq 2000 --steps 1 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "qadc trace" | tail -12
python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c1.csv python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1.log 2>&1
python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 11 -c 2 -o gpurun_out/prof_c1 python bench.py --workload c1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c1_full.log 2>&1
ls -la gpurun_out
