#pragma once
#include <cstdio>

// Debug builds (-DPGSAG_DEBUG_BOUNDS, `tools/debug_checks.sh`): device-side bounds and invariant
// checks on every gathered index, scatter position and shared-memory slot of the path; a failed
// check prints its location and traps (the CUDA call then fails loudly).  They stand in for
// compute-sanitizer, which this GPU pool does not allow.  Compiled out otherwise.
#ifdef PGSAG_DEBUG_BOUNDS
#include <cstdio>
#define PGSAG_DCHECK(c)                                                                 \
  do {                                                                                  \
    if (!(c)) {                                                                         \
      printf("PGSAG_DCHECK failed at %s:%d: %s\n", __FILE__, __LINE__, #c);             \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define PGSAG_DCHECK(c) \
  do {                  \
  } while (0)
#endif

