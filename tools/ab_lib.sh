#!/bin/bash
# A/B library builds on the bench workload in ONE gpurun call (same box):
#   tools/ab_lib.sh path/a.so path/b.so ...   ("" = in-tree build)
for lib in "$@"; do
  for rep in 1 2; do
    TAFV_GPU_LIB=$lib python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ablib.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ablib.json').read().strip().splitlines()[-1])
print('$lib' or 'in-tree', 'rep $rep', round(d['value']/1e6,1), 'Mupd/s', round(d['ms_per_step'],4), 'ms/step')"
  done
done
