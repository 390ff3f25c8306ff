#!/bin/bash
# A/B the library's launch knobs on the bench workload: tools/ab.sh "flagA=1" "flagA=0 flagB=2" ...
mkdir -p gpurun_out
for spec in "$@"; do
  args=""; for f in $spec; do args="$args --flag $f"; done
  tag=$(echo "$spec" | tr ' =' '_-')
  python bench.py --no-cpu-baseline --e2e-steps 1 $args > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python - "$spec" "gpurun_out/ab_$tag.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"[{sys.argv[1]}] {d['value']/1e6:.1f} Mupd/s  {d['ms_per_step']:.3f} ms/step  iter-roofline {d['roofline_iteration']['frac']:.3f}")
for k, v in d["kernels"].items():
    print(f"    {k:16s} {v['ms']:8.3f} ms  {v['GBps']} GB/s")
PY
done
