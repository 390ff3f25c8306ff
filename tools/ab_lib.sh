#!/bin/bash
# A/B library builds on the bench workload in ONE gpurun call (same box):
#   CFG=2 STEPS=20 tools/ab_lib.sh path/a.so path/b.so ...   ("" = in-tree build)
CFG=${CFG:-2}
STEPS=${STEPS:-20}
for rep in 1 2; do
  for lib in "$@"; do
    TAFV_GPU_LIB=$lib python bench.py --config $CFG --steps $STEPS --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      --ensemble 0 > gpurun_out/ablib.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ablib.json').read().strip().splitlines()[-1])
k=d['kernels']
print('${lib:-in-tree}', 'cfg $CFG rep $rep', round(d['value']/1e6,1), 'Mupd/s', round(d['ms_per_step'],4), 'ms/step', ' '.join(f'{n}={v[\"ms\"]:.2f}' for n,v in k.items()))"
  done
done
