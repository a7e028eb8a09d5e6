/* Batched GPU encoder: full-batch Adam fitting of
 * one SIREN per image, the inner loop of encoder._train
 * (encoder.py:66-85) over net.loss_and_grad (net.py:217-265) and net.Adam
 * (net.py:268-300).
 *
 * Models use the transform layout of rinr_b200_transforms.h: d_w [n][P] f32
 * (matrices concatenated, row-major (out, in)), d_b [n][sum dims[1..]] f32,
 * d_mask [n][P] u8.  Architectures: (2, H, H, 3) with 8 <= H <= 16 run the
 * fused narrow kernel (the CIFAR net of PAPER.md:441 is H = 15); any other
 * (2, d1, ..., 3) with widths <= 64 and <= 16 weight matrices (the 10-layer
 * 102flowers / Mini-ImageNet nets) runs the general kernels
 * (fit_general.cu: per Adam step one forward/backward launch over 32-pixel
 * tiles with several CTAs per image and one update launch).
 *
 * Narrow kernel: one CTA fits one image and all `steps` Adam steps of a
 * round run inside one launch, with weights, moments and masks in shared
 * memory.  The arithmetic
 * follows the reference's fp32 algorithm:
 *   * RINR_SIN_ACCURATE: forward / backward per pixel in fp32 FFMA with
 *     accurate sinf, gradient sums in 3xTF32 (fp32-accurate);
 *   * RINR_SIN_MUFU (H < 16): the matrix products and gradient sums on
 *     mma.sync in bf16 3-pass (about 2^-16 relative per product), sines on MUFU;
 *   * the Adam update reproduces numpy's f32 operation order exactly.
 * Gradients match net.loss_and_grad to summation order (tests state
 * the tolerance); trajectories therefore agree statistically, not bitwise.
 */
#ifndef RINR_B200_ENCODER_H
#define RINR_B200_ENCODER_H

#include <stddef.h>
#include <stdint.h>

#include "rinr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t h, w;        /* image size; targets d_images [n][h*w*3] f32 HWC in [0,1] */
  int32_t steps;       /* Adam steps of this round (>= 0)                       */
  int32_t sin_mode;    /* RINR_SIN_MUFU | RINR_SIN_ACCURATE                     */
  double lr0;          /* cosine-decay peak (encoder.py:28-30)                  */
  double omega;        /* arch omega (net.py:21)                                 */
  int32_t curve_cap;   /* doubles per image in d_curve (>= steps/stride + 2)    */
  const float* sched;  /* nullable device [steps][3] f32: per step t the values
                          encoder._train and net.Adam use, f32(cosine_lr(lr0, t,
                          steps)), f32(1 - 0.9**(t+1)), f32(1 - 0.999**(t+1)),
                          computed on the host exactly as Python does; NULL:
                          computed in the kernel (f64 pow / cos)                */
} rinr_fit_params_t;

/* Run `steps` Adam steps per image, updating d_w / d_b in place (masked
 * weights stay exactly 0).  d_curve [n][curve_cap] f64 receives the losses
 * encoder._train samples (every max(1, steps/64)-th step plus the final
 * loss), padded with NaN.  d_status[n]: 0, or t+1 if the loss became
 * non-finite at step t (t == steps for the final loss) -> TrainingError.
 * d_grad_w / d_grad_b (nullable, [n][P] / [n][PB] f32): the gradient of the
 * FIRST step (masked, as net.loss_and_grad returns it), and d_loss0 [n] f64
 * its loss; with steps == 0 nothing is updated (the loss_and_grad parity
 * hook). */
RINR_API int rinr_fit(const int32_t* dims, int nl, int64_t n, float* d_w, float* d_b, const uint8_t* d_mask,
                      const float* d_images, const rinr_fit_params_t* params, double* d_curve, int32_t* d_status,
                      float* d_grad_w, float* d_grad_b, double* d_loss0, void* stream);

/* decoder.decode of the fitted models at their own size: d_out [n][h*w*3]
 * f32 HWC, clipped to [0,1] (for PSNR against the targets). */
RINR_API int rinr_fit_render(const int32_t* dims, int nl, int64_t n, const float* d_w, const float* d_b, int32_t h,
                             int32_t w, double omega, int32_t sin_mode, float* d_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif
