#!/bin/bash
# Full ncu capture of one kernel of the bench workload (run under gpurun):
#   tools/ncu_kernel.sh <regex> <skip> <count> <out-name> [bench flags...]
set -e
mkdir -p gpurun_out
re=$1; skip=$2; count=$3; out=$4; shift 4
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 $*"
$CMD > gpurun_out/${out}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$re" -s $skip -c $count \
    -o gpurun_out/$out $CMD > gpurun_out/${out}_ncu.log 2>&1
echo "captured gpurun_out/$out.ncu-rep"
