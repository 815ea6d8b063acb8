#!/bin/bash
# usage: tools/sweep_build.sh "<nvcc extra flags>" ... : rebuild with each flag set and run a short bench
# (C4, 5 steps of 8 views); prints Mpix/s and the per-view times of the main kernels
for fl in "$@"; do
  PGSAG_NVCC_EXTRA="$fl" python -c "from paper_2501_01677_b200 import build; build.build(force=True)" >/dev/null || exit 1
  python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-train 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels_ms_per_view']
s=lambda p: round(sum(v for n, v in k.items() if n.startswith(p)), 4)
print('$fl', round(d['value'],1), 'A7', s('A7'), 'A6', s('A6'), 'sort(A2-A5)', s('A2')+s('A3')+s('A4')+s('A5'), 'A0', s('A0'))"
done
