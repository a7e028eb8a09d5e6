/* Encoder-side model transforms on the GPU: magnitude pruning, layer-wise
 * affine quantisation and PSNR.
 *
 * Every function works on a batch of n models of ONE architecture
 * dims[0..nl] (nl weight matrices), stored device-resident as
 *   d_w    [n][P] f32   all weight matrices of a model, layer by layer,
 *                       each row-major (out, in); P = sum_l dims[l]*dims[l+1]
 *   d_mask [n][P] u8    1 = kept
 * which is the concatenation order the reference ranks magnitudes in
 * (compressor.py:100-105).  Results are bit-identical to the reference
 * (uint32 compares in tests/test_gpu_transforms.py); PSNR is f64 with a
 * different summation order (relative difference <= 1e-12).
 *
 * Calls are asynchronous on `stream`; per-model failures are reported in
 * d_status[n] (0 = ok, else a RINR_ERR_* code) and never abort the batch.
 */
#ifndef RINR_B200_TRANSFORMS_H
#define RINR_B200_TRANSFORMS_H

#include <stddef.h>
#include <stdint.h>

#include "rinr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

enum { RINR_PRUNE_GLOBAL = 0, RINR_PRUNE_PER_LAYER = 1 };

/* compressor.prune_l1 (compressor.py:108-152): per model, the
 * k = floor(ratio*N + 0.5) smallest |w| (N = P for GLOBAL, per matrix for
 * PER_LAYER; ties by position, already-zero entries counted) lose their mask
 * bit and every weight is multiplied by its mask (negative pruned weights
 * become -0.0).  A model whose new masks would empty a whole matrix keeps its
 * weights and masks and gets d_status = RINR_ERR_STRUCTURAL. */
RINR_API int rinr_prune_l1(const int32_t* dims, int nl, int64_t n, float* d_w, uint8_t* d_mask,
                           const double* d_ratio, int scope, int32_t* d_status, void* stream);

/* compressor.quantize (compressor.py:160-202) of the hidden matrices
 * (1 .. nl-2) with `bits` = 8 or 16, plus quantize_codes (205-218).  Per
 * (model, hidden layer h): d_scale / d_zp / d_const [n][nl-2]; kept weights
 * snapped in place to f32(scale*(code-zp)) * mask; d_codes [n][P] u16
 * receives the codes of every entry of quantised layers (0 elsewhere).
 * A model with a non-finite weight or bias anywhere (d_b: [n][sum dims[1..]]
 * f32, biases layer by layer) is left untouched with d_status =
 * RINR_ERR_NUMERIC. */
RINR_API int rinr_quantize(const int32_t* dims, int nl, int64_t n, int bits, float* d_w, const uint8_t* d_mask,
                           const float* d_b, double* d_scale, int32_t* d_zp, uint8_t* d_const, uint16_t* d_codes,
                           int32_t* d_status, void* stream);

/* metrics.psnr (metrics.py:23-41) for n image pairs of `count` values each
 * (f32 in [0,1]); quantized != 0 rounds both through u8 first (image.py:49-55).
 * d_mse[n] f64; d_psnr[n] f64 (+inf when equal). */
RINR_API int rinr_psnr(const float* d_a, const float* d_b, int64_t n, int64_t count, int quantized, double* d_mse,
                       double* d_psnr, void* stream);

#ifdef __cplusplus
}
#endif

#endif
