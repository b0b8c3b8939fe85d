// check.cuh -- device-side bounds assertions of the CHECKED build (EH_CHECKED).
//
// compute-sanitizer is closed on this GPU pool, so the test suite instead runs a
// build of the library compiled with -DEH_CHECKED (lib/libeh_checked.so, see
// build.py) in which every EH_DASSERT below is live: a violated bound prints the
// condition and its source line and traps the kernel (the launch fails, the call
// returns EH_ECUDA).  In the product build the macro compiles to nothing.
#pragma once
#include <cstdio>

#ifdef EH_CHECKED
#define EH_DASSERT(c)                                                                              \
  do {                                                                                             \
    if (!(c)) {                                                                                    \
      printf("EH_DASSERT failed: %s (%s:%d, block %d thread %d)\n", #c, __FILE__, __LINE__,        \
             (int)blockIdx.x, (int)threadIdx.x);                                                   \
      __trap();                                                                                    \
    }                                                                                              \
  } while (0)
#else
#define EH_DASSERT(c) \
  do {                \
  } while (0)
#endif
