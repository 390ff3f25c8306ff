#!/bin/bash
# Per-kernel breakdown for several library builds (timing experiments).
for lib in "$@"; do
  TAFV_GPU_LIB=$lib python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/ablibk.json 2>/dev/null
  python - "$lib" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ablibk.json").read().strip().splitlines()[-1])
print(f"[{sys.argv[1] or 'in-tree'}] {d['value']/1e6:.1f} Mupd/s {d['ms_per_step']:.3f} ms/step")
for k, v in d["kernels"].items():
    print(f"    {k:16s} {v['ms']:8.3f} ms")
PY
done
