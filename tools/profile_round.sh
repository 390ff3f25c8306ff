#!/bin/bash
# Round profiling evidence (run under gpurun, one GPU), on one steady-state
# iteration of a config (tools/prof_region.py brackets it with
# cudaProfilerStart/Stop, so mesh build and graph capture are not profiled):
#   1. plain run of the profiled command (must exit 0 first)
#   2. ncu launch list: duration + DRAM bytes of every launch of the iteration
#   3. ncu --set full of the first launch of K1, K2 and K3 (the top-level phase)
#   tools/profile_round.sh <tag> [config]      e.g.  tools/profile_round.sh r2cfg4 4
# Outputs in gpurun_out/; summarise with tools/summarize_ncu.py <tag> into profiles/.
set -e
tag=${1:-r2}
CFG=${2:-4}
mkdir -p gpurun_out
CMD="python tools/prof_region.py --config $CFG --warmup 2 --iters 1"
$CMD > gpurun_out/prof_${tag}_plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv $CMD > /dev/null 2>&1
for k in k_grad_limit k_face_flux k_gather_update; do
  ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/full_${tag}_$k $CMD > /dev/null 2>&1
done
echo done
