#!/bin/bash
# Debug build with the device-side bounds / invariant checks (-DPGSAG_DEBUG_BOUNDS, internal.cuh), then the
# sanitizer workload (tools/sanitize_run.py: C1 and a C2-shaped scene through A0-A8, both sort paths, one training
# iteration with densification) and the randomised parity sweep on it.  Any failed check traps the kernel and fails
# the run.  The release build is restored at the end.
set -e
PGSAG_NVCC_EXTRA="-DPGSAG_DEBUG_BOUNDS" python -c "from paper_2501_01677_b200 import build; build.build(force=True)"
python tools/sanitize_run.py
PGSAG_FUZZ_SEEDS=${SEEDS:-256} python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py -q -x -p no:cacheprovider
python tools/debug_negative.py  # the checks themselves must catch a corrupted sort entry
python -c "from paper_2501_01677_b200 import build; build.build(force=True)"
