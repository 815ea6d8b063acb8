#!/bin/bash
# usage: tools/ncu_variant.sh <tag> "<nvcc extra flags>" <kernel regex> : rebuild with the flags and capture the
# kernel once (ncu --set full, one C4 view) into gpurun_out/<tag>.ncu-rep
tag=$1; fl=$2; kre=$3
PGSAG_NVCC_EXTRA="$fl" python -c "from paper_2501_01677_b200 import build; build.build(force=True)" >/dev/null || exit 1
python tools/profile_step.py --steps 1 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -c 1 -o gpurun_out/$tag \
  python tools/profile_step.py --steps 1 > gpurun_out/$tag.log 2>&1
