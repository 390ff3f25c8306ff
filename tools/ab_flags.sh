#!/bin/bash
# A/B library flags on one config in ONE gpurun call (same box), each flag set
# run twice, interleaved:
#   CFG=4 STEPS=5 tools/ab_flags.sh "" "slot_geo=0" "slot_n=0" ...
# ("" = defaults; several flags: "a=0,b=1")
CFG=${CFG:-3}
STEPS=${STEPS:-5}
for rep in 1 2; do
  for fl in "$@"; do
    args=""
    for kv in ${fl//,/ }; do args="$args --flag $kv"; done
    python bench.py --config $CFG --steps $STEPS --warmup 3 --no-cpu-baseline --e2e-steps 1 --ensemble 0 $args \
      > gpurun_out/abflag.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/abflag.json').read().strip().splitlines()[-1])
k=d['kernels']
print('[${fl:-default}]', 'cfg $CFG rep $rep', round(d['value']/1e6,1), 'Mupd/s', round(d['ms_per_step'],3), 'ms/step', ' '.join(f'{n}={v[\"ms\"]:.2f}' for n,v in k.items()))"
  done
done
