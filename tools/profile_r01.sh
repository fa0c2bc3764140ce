#!/bin/bash
# Profile capture (run under gpurun): launch list + full captures of the dominant scan kernel,
# each only after the identical command exited 0 without ncu.   usage: tools_profile.sh <tag>
TAG=${1:-r01}
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qadc|scan_kernel|pack_tiles|flat_tables|seed_topk|tighten|finalize|init_select" -c 400 --csv --log-file gpurun_out/${TAG}_launches_c2.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
$CMD > gpurun_out/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 15 -c 1 -o gpurun_out/${TAG}_scan_c2 $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
for W in c1 c3; do
CMDW="python bench.py --workload $W --steps 2 --warmup 3 --no-cpu-baseline"
S=11; [ $W = c3 ] && S=15
$CMDW > gpurun_out/${TAG}_plain_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s $S -c 1 -o gpurun_out/${TAG}_scan_$W $CMDW > gpurun_out/${TAG}_ncu_full_$W.log 2>&1
done
CMD5="python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline"
$CMD5 > gpurun_out/${TAG}_plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ivf_|probe_|scan_kernel|tighten|pack_tiles|finalize|init_select|seed" -s 1 -c 34 --csv --log-file gpurun_out/${TAG}_launches_c5.csv $CMD5 > gpurun_out/${TAG}_ncu_c5.log 2>&1
$CMD5 > gpurun_out/${TAG}_plain_c5b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 6 -c 1 -o gpurun_out/${TAG}_scan_c5 $CMD5 > gpurun_out/${TAG}_ncu_full_c5.log 2>&1
ls -la gpurun_out | grep ${TAG}_ | tail -20
# summaries are produced here (the .ncu-rep files together exceed what gpurun copies back) and the reports dropped
python tools/summarize_profiles.py ${TAG} && mkdir -p gpurun_out/${TAG}_summaries && cp profiles/${TAG}_* gpurun_out/${TAG}_summaries/
rm -f gpurun_out/${TAG}_scan_*.ncu-rep
