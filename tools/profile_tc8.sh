#!/bin/bash
# ncu capture of the tensor-core scan kernel on a shortened C4 (run under gpurun).  usage: tools/profile_tc8.sh <tag>
TAG=${1:-r02_tc8}
CMD="python bench.py --workload c4 --n 40000000 --nq 2560 --steps 1 --warmup 3 --also '' --no-cpu-baseline --no-parity --option force_variant=12"
eval $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_tc8 -s 8 -c 1 -o gpurun_out/${TAG} bash -c "$CMD" > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
ls -la gpurun_out/${TAG}*
