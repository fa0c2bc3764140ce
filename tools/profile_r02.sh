#!/bin/bash
# Round-2 profile capture (run under gpurun): launch lists + full captures of the dominant kernels, each only after
# the identical command exited 0 without ncu.   usage: tools/profile_r02.sh [tag]
TAG=${1:-r02}
ONLY=${2:-all}   # all | c4 | c5
LIB='qadc|scan_|pack_tiles|flat_tables|seed_topk|tighten|finalize|init_select|probe_|ivf_'
C4="python bench.py --workload c4 --steps 1 --warmup 3 --also '' --no-cpu-baseline --no-parity"
C5="python bench.py --workload c5g --steps 1 --warmup 3 --also '' --no-cpu-baseline --no-parity"
if [ "$ONLY" != "c5" ]; then
# C4 (the headline): every library launch of the first step (15 segments), then the 6.7e7-code segment of the tensor-core scan in full
eval $C4 > gpurun_out/${TAG}_plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$LIB" -c 40 --csv --log-file gpurun_out/${TAG}_launches_c4.csv bash -c "$C4" > gpurun_out/${TAG}_ncu_launch_c4.log 2>&1
eval $C4 > gpurun_out/${TAG}_plain_c4b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:scan_tc8 -s 13 -c 1 -o gpurun_out/${TAG}_scan_c4 bash -c "$C4" > gpurun_out/${TAG}_ncu_full_c4.log 2>&1
fi
if [ "$ONLY" != "c4" ]; then
# C5 (IVF): launch list of one step, the first scan round and the probe contraction in full
eval $C5 > gpurun_out/${TAG}_plain_c5.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$LIB" -s 1 -c 40 --csv --log-file gpurun_out/${TAG}_launches_c5.csv bash -c "$C5" > gpurun_out/${TAG}_ncu_launch_c5.log 2>&1
eval $C5 > gpurun_out/${TAG}_plain_c5b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"scan_kernel" -s 6 -c 1 -o gpurun_out/${TAG}_scan_c5 bash -c "$C5" > gpurun_out/${TAG}_ncu_full_c5.log 2>&1
eval $C5 > gpurun_out/${TAG}_plain_c5c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"probe_approx_umma" -s 6 -c 2 -o gpurun_out/${TAG}_probe_c5 bash -c "$C5" > gpurun_out/${TAG}_ncu_full_probe.log 2>&1
fi
python tools/summarize_profiles.py ${TAG} && mkdir -p gpurun_out/${TAG}_summaries && cp profiles/${TAG}_* gpurun_out/${TAG}_summaries/
ls -la gpurun_out | grep ${TAG}_ | tail -20
rm -f gpurun_out/${TAG}_scan_*.ncu-rep gpurun_out/${TAG}_probe_*.ncu-rep
