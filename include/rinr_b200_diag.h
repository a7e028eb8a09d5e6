/*
 * rinr_b200_diag.h — measurement-only entry points of librinr_b200.so (not part
 * of the decode ABI and with no reference counterpart).  bench.py uses them to
 * measure the pipe peaks its roofline fractions divide by.
 */
#ifndef RINR_B200_DIAG_H
#define RINR_B200_DIAG_H

#include "rinr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

enum rinr_diag_kind { RINR_DIAG_MUFU_SIN = 0, RINR_DIAG_FFMA = 1, RINR_DIAG_HMMA_BF16 = 2 };

/* Launch one pipe-saturating microbenchmark kernel on `stream` (no sync);
 * *ops_per_launch receives the operation count (sines or flops) it performs. */
RINR_API int rinr_diag_launch(int kind, int blocks, int threads, int iters, float* d_sink, void* stream,
                              double* ops_per_launch);

#ifdef __cplusplus
}
#endif

#endif /* RINR_B200_DIAG_H */
