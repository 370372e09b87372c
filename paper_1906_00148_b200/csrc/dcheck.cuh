// dcheck.cuh — device-side bounds checks of the checked build (-DSHE_CHECKED,
// tools/gpu_checked.sh).  compute-sanitizer is closed on this GPU pool
// (profiles/r2b/compute_sanitizer_racecheck_r2.log), so the default path's
// runtime-computed indices (TMEM columns and lanes, shared-memory slots,
// lane-list and gate indices, key-switch tiles) are asserted instead; a
// failed check prints its site and traps (the launch fails, the host call
// returns SHE_ERR_CUDA).  In the product build the checks compile to nothing.
#pragma once
#include <stdio.h>
#ifdef SHE_CHECKED
#define SHE_DCHECK(cond)                                                                        \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("SHE_DCHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define SHE_DCHECK(cond) ((void)0)
#endif
