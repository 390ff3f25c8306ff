#!/bin/bash
# Brick K1 variants (library builds with different stage sizes) on one config, each with k1_brick=1:
#   CFG=4 STEPS=5 tools/ab_brick.sh ablibs/a.so ablibs/b.so ...
CFG=${CFG:-4}
STEPS=${STEPS:-5}
for rep in 1 2; do
  for lib in "$@"; do
    TAFV_GPU_LIB=$lib python bench.py --config $CFG --steps $STEPS --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      --ensemble 0 --flag k1_brick=1 > gpurun_out/abbrick.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abbrick.json').read().strip().splitlines()[-1])
k=d['kernels']
print('$lib', 'cfg $CFG rep $rep', round(d['value']/1e6,1), 'Mupd/s', round(d['ms_per_step'],3), 'ms/step', 'K1', round(k['K1_grad_limit']['ms'],1))"
  done
done
