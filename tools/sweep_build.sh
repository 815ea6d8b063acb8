#!/bin/bash
# usage: tools/sweep_build.sh "<nvcc extra flags>" ... : rebuild with each flag set and run a short bench
for fl in "$@"; do
  PGSAG_NVCC_EXTRA="$fl" python -c "from paper_2501_01677_b200 import build; build.build(force=True)" >/dev/null || exit 1
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-train 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_step']
print('$fl', round(d['value'],1), 'A7', k.get('A7_render_bwd'), 'A6', k.get('A6_render_fwd'))"
done
