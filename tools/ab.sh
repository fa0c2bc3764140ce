#!/bin/bash
# A/B helper: tools_ab.sh <workload> <extra bench args...>   prints per-segment scan times and value
wl=$1; shift
QADC_TRACE=1 python bench.py --workload $wl --steps 1 --warmup 3 --no-cpu-baseline "$@" 2>&1 | grep -E "qadc trace|\"value\"" | tail -9 | sed -E 's/\{"metric.*"value": ([0-9.e+]+).*"ms_per_step": ([0-9.]+).*/VALUE \1 ms_per_step \2/' | grep -E "stage 1|VALUE"
