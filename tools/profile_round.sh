#!/bin/bash
# Round profiling evidence (run under gpurun, one GPU):
#   1. plain run of the profiled bench command (must exit 0 first)
#   2. ncu launch list (gpu__time_duration of every launch)
#   3. ncu --set full of one iteration's worth (8 launches for theta=2) of K1, K2, K3
# PROFILE_CMD / PROFILE_COUNT override the profiled command / launches per kernel.
# Outputs in gpurun_out/; summarise with tools/summarize_ncu.py into profiles/.
set -e
tag=${1:-r1}
mkdir -p gpurun_out
CMD=${PROFILE_CMD:-"python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1"}
NC=${PROFILE_COUNT:-8}
$CMD > gpurun_out/prof_${tag}_plain.json 2> gpurun_out/prof_${tag}_plain.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}.csv $CMD > /dev/null 2>&1
for k in k_grad_limit k_face_flux k_gather_update; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c $NC \
      -o gpurun_out/full_${tag}_$k $CMD > /dev/null 2>&1
done
echo done
