// General-architecture GPU encoder (SURVEY.md §8(f) rank 1 beyond the CIFAR
// net): full-batch Adam fitting of one SIREN per image for ANY architecture
// (2, d1, ..., d_{L-1}, 3) with widths <= 64 and <= 16 weight matrices —
// e.g. the paper's 10-layer [2,32x9,3] (102flowers) and [2,40x9,3]
// (Mini-ImageNet) nets.  Same C ABI as the narrow kernel
// (rinr_fit / rinr_fit_render dispatch here when the architecture is not
// (2, H, H, 3) with 8 <= H <= 16).
//
// Per Adam step of a round, two launches (the host issues steps + 1 pairs):
//   gen_grad_kernel  grid (CTAs per image, n): each CTA runs forward +
//                    backward for 32-pixel tiles of its image with the
//                    weights in shared memory (net.loss_and_grad,
//                    net.py:217-265: z = a @ W^T + b, a = sin(omega z), MSE
//                    mean over 3P values, delta = (2/3P) resid,
//                    delta_{l-1} = (delta W) * omega cos(omega z)); it sums
//                    the tile's weight / bias gradients (Delta^T A over the
//                    pixels) into shared accumulators and adds them to the
//                    image's global gradient with one atomicAdd per entry,
//                    plus the f64 loss.
//   gen_adam_kernel  grid (n): loss check / curve sample (encoder._train,
//                    encoder.py:66-85), then net.Adam.step (net.py:282-296)
//                    in numpy's f32 operation order with the host schedule
//                    table, masks re-applied; zeroes the gradient for the
//                    next step.
// fp32 FFMA throughout; sines accurate (sinf / cosf) or MUFU (__sinf /
// __cosf).  Gradient sums differ from numpy's BLAS in summation order (and
// atomics make them order-nondeterministic), so trajectories agree with the
// reference statistically; tests state the tolerance.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/rinr_b200_encoder.h"
#include "device_common.cuh"

namespace rinr {
namespace {

constexpr int kGMaxL = 16;   // weight matrices
constexpr int kGMaxW = 64;   // widths
constexpr int kTile = 32;    // pixels per tile
constexpr int kGThreads = 256;
constexpr int kGroups = kGThreads / 32;          // pixel-lane groups (warps)
constexpr int kPerT = (kGMaxW + kGroups - 1) / kGroups;  // outputs per thread (register tile)

struct GArch {
  int nl;
  int dims[kGMaxL + 1];
  int woff[kGMaxL];  // weight offset of matrix l in [P]
  int boff[kGMaxL];  // bias offset of layer l in [PB]
  int P, PB, maxw;
};

struct GArgs {
  GArch A;
  int64_t n;
  const float* images;
  int h, wd, hw;
  double inv_wm1, inv_hm1;
  float omega;
  int acc;  // accurate sine
  int ctas_per_image;
};

__device__ __forceinline__ void gsincos(bool acc, float x, float& s, float& c) {
  if (acc) sincosf(x, &s, &c);
  else {
    s = __sinf(x);
    c = __cosf(x);
  }
}

// Shared-memory map of the gradient kernel (floats):
//   ws  [P + PB]         weights then biases
//   gacc[P + PB]         this CTA's gradient sums
//   z   [nl-1][maxw][32] hidden pre-activations of the tile (omega*z kept)
//   act [2][maxw][32]    current layer input / delta ping-pong
//   d2  [2][maxw][32]    deltas ping-pong
__host__ __device__ inline size_t gen_smem_floats(const GArch& A) {
  return size_t(2) * (A.P + A.PB) + size_t(A.nl - 1) * A.maxw * kTile + size_t(4) * A.maxw * kTile + 64;
}

// z_out[o][px] = sum_i W[o][i] in[i][px] + b[o] for one tile.  Thread ->
// (px = t % 32, outputs o = t/32 + 8k): each input activation is loaded once
// and reused for the thread's kPerT outputs (register tile).
__device__ __forceinline__ void tile_linear(const float* W, const float* b, int fi, int fo, const float* in,
                                            float* out, int tid) {
  const int px = tid & 31, og = tid >> 5;
  float z[kPerT];
#pragma unroll
  for (int k = 0; k < kPerT; ++k) z[k] = 0.0f;
  for (int i = 0; i < fi; ++i) {
    const float a = in[i * kTile + px];
#pragma unroll
    for (int k = 0; k < kPerT; ++k) {
      const int o = og + kGroups * k;
      if (o < fo) z[k] = fmaf(a, W[o * fi + i], z[k]);
    }
  }
#pragma unroll
  for (int k = 0; k < kPerT; ++k) {
    const int o = og + kGroups * k;
    if (o < fo) out[o * kTile + px] = __fadd_rn(z[k], b[o]);
  }
}

// gW[o][i] += sum_q delta[o][q] a[i][q] and gb[o] += sum_q delta[o][q] over
// the tile, with 2 x 4 register tiles of (o, i) per thread.
__device__ __forceinline__ void tile_grads(const float* dcur, const float* ain, int fi, int fo, float* gw, float* gb,
                                           int tid) {
  const int nib = (fi + 3) / 4, ntile = ((fo + 1) / 2) * nib;
  for (int t = tid; t < ntile; t += kGThreads) {
    const int o0 = 2 * (t / nib), i0 = 4 * (t - (t / nib) * nib);
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    for (int q = 0; q < kTile; ++q) {
      const float d0 = dcur[o0 * kTile + q], d1 = o0 + 1 < fo ? dcur[(o0 + 1) * kTile + q] : 0.0f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float a = i0 + c < fi ? ain[(i0 + c) * kTile + q] : 0.0f;
        acc[0][c] = fmaf(d0, a, acc[0][c]);
        acc[1][c] = fmaf(d1, a, acc[1][c]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (o0 + r < fo && i0 + c < fi) gw[(o0 + r) * fi + i0 + c] = __fadd_rn(gw[(o0 + r) * fi + i0 + c], acc[r][c]);
  }
  for (int o = tid; o < fo; o += kGThreads) {
    float sacc = 0.0f;
    for (int q = 0; q < kTile; ++q) sacc = __fadd_rn(sacc, dcur[o * kTile + q]);
    gb[o] = __fadd_rn(gb[o], sacc);
  }
}

__global__ void __launch_bounds__(kGThreads) gen_grad_kernel(GArgs g, const float* __restrict__ w,
                                                             const float* __restrict__ b, float* __restrict__ grad,
                                                             double* __restrict__ loss, const int32_t* status) {
  extern __shared__ __align__(16) float sm[];
  const GArch& A = g.A;
  const int64_t m = blockIdx.y;
  if (status[m]) return;  // this image already failed
  const int tid = threadIdx.x, px = tid & 31;
  const int NP = A.P + A.PB;
  float* ws = sm;
  float* gacc = ws + NP;
  float* zb = gacc + NP;
  float* act = zb + (A.nl - 1) * A.maxw * kTile;
  float* dl = act + 2 * A.maxw * kTile;
  for (int p = tid; p < NP; p += kGThreads) {
    ws[p] = p < A.P ? w[m * A.P + p] : b[m * A.PB + p - A.P];
    gacc[p] = 0.0f;
  }
  __syncthreads();
  const float om = g.omega;
  const int ntile = (g.hw + kTile - 1) / kTile;
  double lsum = 0.0;
  const float dscale = float(2.0 / (3.0 * double(g.hw)));  // (2.0 * scale) as numpy's weak scalar
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int p = tile * kTile + px;
    const bool inside = p < g.hw;
    // ---- forward (net.py:183-202) ----
    if (tid < kTile) {
      const int pr = inside ? p / g.wd : 0, pc = inside ? p - pr * g.wd : 0;
      act[0 * kTile + px] = grid_coord(pc, g.wd, g.inv_wm1);
      act[1 * kTile + px] = grid_coord(pr, g.h, g.inv_hm1);
    }
    __syncthreads();
    float* in = act;
    float* nxt = act + A.maxw * kTile;
    for (int l = 0; l < A.nl; ++l) {
      const int fi = A.dims[l], fo = A.dims[l + 1];
      const bool last = l == A.nl - 1;
      float* zo = last ? nxt : zb + l * A.maxw * kTile;
      tile_linear(ws + A.woff[l], ws + A.P + A.boff[l], fi, fo, in, zo, tid);
      __syncthreads();
      if (!last) {
        for (int e = tid; e < fo * kTile; e += kGThreads) {
          const float wz = __fmul_rn(om, zo[e]);  // np.sin(omega * z) in f32
          float s, c;
          gsincos(g.acc, wz, s, c);
          nxt[e] = s;
          zo[e] = wz;  // keep omega*z for the backward cosine
        }
        __syncthreads();
        float* t = in;
        in = nxt;
        nxt = t;
      }
    }
    // nxt holds the output layer [3][32]; in holds the last hidden activations
    // ---- loss and output delta ----
    float* dcur = dl;
    if (tid < 3 * kTile) {
      const int j = tid / kTile, q = tid % kTile, pp = tile * kTile + q;
      float r = 0.0f;
      if (pp < g.hw) r = __fsub_rn(nxt[j * kTile + q], g.images[(m * g.hw + pp) * 3 + j]);
      lsum += double(r) * double(r);
      dcur[j * kTile + q] = __fmul_rn(dscale, r);  // zero for pixels past the image
    }
    __syncthreads();
    // ---- backward (net.py:250-264) ----
    for (int l = A.nl - 1; l >= 0; --l) {
      const int fi = A.dims[l], fo = A.dims[l + 1];
      // layer input activations a_{l-1}: recompute sin from the stored omega*z
      const float* ain;
      float* abuf = act;  // free now: reuse as the activation buffer
      if (l == 0) {
        if (tid < kTile) {
          const int p0 = tile * kTile + px;
          const int pr = p0 < g.hw ? p0 / g.wd : 0, pc = p0 < g.hw ? p0 - pr * g.wd : 0;
          abuf[0 * kTile + px] = grid_coord(pc, g.wd, g.inv_wm1);
          abuf[1 * kTile + px] = grid_coord(pr, g.h, g.inv_hm1);
        }
      } else {
        const float* zl = zb + (l - 1) * A.maxw * kTile;
        for (int e = tid; e < fi * kTile; e += kGThreads) {
          float s, c;
          gsincos(g.acc, zl[e], s, c);
          abuf[e] = s;
        }
      }
      ain = abuf;
      __syncthreads();
      // gW[o][i] += sum_px delta[o][px] a[i][px];  gb[o] += sum_px delta[o][px]
      tile_grads(dcur, ain, fi, fo, gacc + A.woff[l], gacc + A.P + A.boff[l], tid);
      if (l > 0) {
        // delta_{l-1}[i] = (sum_o delta[o] W[o][i]) * omega cos(omega z_{l-1}[i])
        float* dn = dcur == dl ? dl + A.maxw * kTile : dl;
        const float* W = ws + A.woff[l];
        const float* zl = zb + (l - 1) * A.maxw * kTile;
        const int ig = tid >> 5;
        float sacc[kPerT];
#pragma unroll
        for (int k = 0; k < kPerT; ++k) sacc[k] = 0.0f;
        for (int o = 0; o < fo; ++o) {
          const float d = dcur[o * kTile + px];
#pragma unroll
          for (int k = 0; k < kPerT; ++k) {
            const int i = ig + kGroups * k;
            if (i < fi) sacc[k] = fmaf(d, W[o * fi + i], sacc[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < kPerT; ++k) {
          const int i = ig + kGroups * k;
          if (i < fi) {
            float s, c;
            gsincos(g.acc, zl[i * kTile + px], s, c);
            dn[i * kTile + px] = __fmul_rn(sacc[k], __fmul_rn(om, c));
          }
        }
        __syncthreads();
        dcur = dn;
      }
      __syncthreads();
    }
  }
  // ---- flush: one atomic per gradient entry, f64 loss ----
  for (int p = tid; p < NP; p += kGThreads) atomicAdd(grad + m * NP + p, gacc[p]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, d);
  __shared__ double red[kGThreads / 32];
  if ((tid & 31) == 0) red[tid >> 5] = lsum;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < kGThreads / 32; ++i) t += red[i];
    atomicAdd(loss + m, t);
  }
}

struct GStep {
  int t, steps, cap, stride;
  const float* sched;
  double lr0;
};

__global__ void __launch_bounds__(256) gen_adam_kernel(GArgs g, GStep s, float* __restrict__ w, float* __restrict__ b,
                                                       const uint8_t* __restrict__ mask, float* __restrict__ grad,
                                                       float* __restrict__ mom, float* __restrict__ vel,
                                                       double* __restrict__ loss, double* __restrict__ curve,
                                                       int32_t* __restrict__ status, int32_t* __restrict__ slots,
                                                       float* __restrict__ grad_w, float* __restrict__ grad_b,
                                                       double* __restrict__ loss0) {
  const GArch& A = g.A;
  const int64_t m = blockIdx.x;
  const int tid = threadIdx.x;
  const int NP = A.P + A.PB;
  float* gr = grad + m * NP;
  __shared__ int s_stop;
  if (tid == 0) {
    s_stop = 0;
    if (!status[m]) {
      const double L = loss[m] / (3.0 * double(g.hw));  // reduction="mean" (net.py:245-247)
      if (!isfinite(L)) {
        status[m] = s.t + 1;  // TrainingError at step t
        s_stop = 1;
      } else if ((s.t % s.stride == 0 || s.t == s.steps) && slots[m] < s.cap) {
        curve[m * s.cap + slots[m]++] = L;
      }
      if (s.t == 0 && loss0) loss0[m] = L;
    } else {
      s_stop = 1;
    }
    loss[m] = 0.0;
  }
  __syncthreads();
  const bool update = !s_stop && s.t < s.steps;
  float lr = 0.f, c1 = 1.f, c2 = 1.f;
  if (update) {
    if (s.sched) {
      lr = s.sched[3 * s.t];
      c1 = s.sched[3 * s.t + 1];
      c2 = s.sched[3 * s.t + 2];
    } else {
      c1 = float(1.0 - pow(0.9, double(s.t + 1)));
      c2 = float(1.0 - pow(0.999, double(s.t + 1)));
      lr = float(0.5 * s.lr0 * (1.0 + cos(3.141592653589793 * double(s.t) / double(s.steps))));
    }
  }
  for (int p = tid; p < NP; p += 256) {
    float gv = gr[p];
    gr[p] = 0.0f;
    const bool isw = p < A.P;
    const float mk = isw ? float(mask[m * A.P + p]) : 1.0f;
    if (isw) gv = __fmul_rn(gv, mk);  // gw * mask (net.py:257)
    if (s.t == 0 && grad_w && !status[m]) {
      if (isw) grad_w[m * A.P + p] = gv;
      else grad_b[m * A.PB + p - A.P] = gv;
    }
    if (!update) continue;
    float* pp = isw ? w + m * A.P + p : b + m * A.PB + (p - A.P);
    const float mp = __fadd_rn(__fmul_rn(mom[m * NP + p], 0.9f), __fmul_rn(float(1.0 - 0.9), gv));
    const float vp = __fadd_rn(__fmul_rn(vel[m * NP + p], 0.999f), __fmul_rn(__fmul_rn(float(1.0 - 0.999), gv), gv));
    mom[m * NP + p] = mp;
    vel[m * NP + p] = vp;
    const float upd = __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mp, c1)), __fadd_rn(__fsqrt_rn(__fdiv_rn(vp, c2)), 1e-8f));
    float nv = __fsub_rn(*pp, upd);
    if (isw) nv = __fmul_rn(nv, mk);  // np.multiply(layer.w, mask)
    *pp = nv;
  }
}

__global__ void gen_pad_kernel(double* curve, const int32_t* slots, int cap) {
  const int64_t m = blockIdx.x;
  for (int s = slots[m] + int(threadIdx.x); s < cap; s += blockDim.x) curve[m * cap + s] = NAN;
}

__global__ void __launch_bounds__(kGThreads) gen_render_kernel(GArgs g, const float* __restrict__ w,
                                                               const float* __restrict__ b, float* __restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  const GArch& A = g.A;
  const int64_t m = blockIdx.y;
  const int tid = threadIdx.x, px = tid & 31;
  const int NP = A.P + A.PB;
  float* ws = sm;
  float* act = ws + NP;
  for (int p = tid; p < NP; p += kGThreads) ws[p] = p < A.P ? w[m * A.P + p] : b[m * A.PB + p - A.P];
  __syncthreads();
  const int ntile = (g.hw + kTile - 1) / kTile;
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int p = tile * kTile + px;
    if (tid < kTile) {
      const int pr = p < g.hw ? p / g.wd : 0, pc = p < g.hw ? p - pr * g.wd : 0;
      act[0 * kTile + px] = grid_coord(pc, g.wd, g.inv_wm1);
      act[1 * kTile + px] = grid_coord(pr, g.h, g.inv_hm1);
    }
    __syncthreads();
    float* in = act;
    float* nxt = act + A.maxw * kTile;
    for (int l = 0; l < A.nl; ++l) {
      tile_linear(ws + A.woff[l], ws + A.P + A.boff[l], A.dims[l], A.dims[l + 1], in, nxt, tid);
      __syncthreads();
      if (l < A.nl - 1) {
        for (int e = tid; e < A.dims[l + 1] * kTile; e += kGThreads) {
          float s, c;
          gsincos(g.acc, __fmul_rn(g.omega, nxt[e]), s, c);
          nxt[e] = s;
        }
        __syncthreads();
      }
      float* t = in;
      in = nxt;
      nxt = t;
    }
    if (tid < 3 * kTile) {
      const int j = tid / kTile, q = tid % kTile, pp = tile * kTile + q;
      if (pp < g.hw) out[(m * g.hw + pp) * 3 + j] = fminf(fmaxf(in[j * kTile + q], 0.0f), 1.0f);
    }
    __syncthreads();
  }
}

int garch_of(const int32_t* dims, int nl, GArch& A) {
  if (!dims || nl < 1 || nl > kGMaxL) return set_error(RINR_ERR_UNSUPPORTED, "GPU encoder: 1..16 weight matrices");
  if (dims[0] != 2 || dims[nl] != 3) return set_error(RINR_ERR_INVALID_INPUT, "architecture must map 2 -> 3");
  A.nl = nl;
  A.P = A.PB = A.maxw = 0;
  for (int l = 0; l <= nl; ++l) {
    if (dims[l] < 1 || dims[l] > kGMaxW) return set_error(RINR_ERR_UNSUPPORTED, "GPU encoder: widths 1..64");
    A.dims[l] = dims[l];
    A.maxw = std::max(A.maxw, dims[l]);
  }
  for (int l = 0; l < nl; ++l) {
    A.woff[l] = A.P;
    A.boff[l] = A.PB;
    A.P += dims[l] * dims[l + 1];
    A.PB += dims[l + 1];
  }
  if (gen_smem_floats(A) * 4 > 226 * 1024) return set_error(RINR_ERR_UNSUPPORTED, "GPU encoder: architecture too large");
  return RINR_OK;
}

int sm_count() {
  int d = 0, v = 148;
  if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
  return v > 0 ? v : 148;
}

GArgs make_gargs(const GArch& A, int64_t n, const float* images, int h, int wd, double omega, int acc) {
  GArgs g{};
  g.A = A;
  g.n = n;
  g.images = images;
  g.h = h;
  g.wd = wd;
  g.hw = h * wd;
  g.inv_wm1 = wd > 1 ? 1.0 / double(wd - 1) : 0.0;
  g.inv_hm1 = h > 1 ? 1.0 / double(h - 1) : 0.0;
  g.omega = float(omega);
  g.acc = acc;
  const int ntile = (g.hw + kTile - 1) / kTile;
  // enough CTAs to cover the GPU twice over, never more than the tiles
  g.ctas_per_image = int(std::max<int64_t>(1, std::min<int64_t>(ntile, (2 * int64_t(sm_count()) + n - 1) / n)));
  return g;
}

int cuda_err(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RINR_OK : set_error(RINR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace
}  // namespace rinr

using namespace rinr;

// Called by rinr_fit (fit.cu) for architectures the narrow kernel does not cover.
int rinr_fit_general(const int32_t* dims, int nl, int64_t n, float* d_w, float* d_b, const uint8_t* d_mask,
                     const float* d_images, const rinr_fit_params_t* p, double* d_curve, int32_t* d_status,
                     float* d_grad_w, float* d_grad_b, double* d_loss0, void* stream) {
  GArch A{};
  if (int e = garch_of(dims, nl, A)) return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const GArgs g = make_gargs(A, n, d_images, p->h, p->w, p->omega, p->sin_mode == RINR_SIN_ACCURATE);
  const size_t NP = size_t(A.P + A.PB);
  // workspace: gradient, moments, f64 loss, curve slots (one allocation, freed at the end)
  void* ws = nullptr;
  const size_t bytes = size_t(n) * NP * 4 * 3 + size_t(n) * 8 + size_t(n) * 4;
  if (cudaMallocAsync(&ws, bytes, st) != cudaSuccess) {
    cudaGetLastError();
    return set_error(RINR_ERR_OOM, "GPU encoder workspace");
  }
  double* loss = static_cast<double*>(ws);  // f64 first: 8-byte aligned whatever n * NP is
  float* grad = reinterpret_cast<float*>(loss + n);
  float* mom = grad + n * NP;
  float* vel = mom + n * NP;
  int32_t* slots = reinterpret_cast<int32_t*>(vel + n * NP);
  if (cudaMemsetAsync(ws, 0, bytes, st) != cudaSuccess || cudaMemsetAsync(d_status, 0, size_t(n) * 4, st) != cudaSuccess)
    return set_error(RINR_ERR_CUDA, "GPU encoder workspace reset");
  const size_t smem = gen_smem_floats(A) * 4;
  // (per call: the attribute is per device and cheap to set)
  if (cudaFuncSetAttribute(gen_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return set_error(RINR_ERR_CUDA, "encoder smem attribute");
  GStep s{};
  s.steps = p->steps;
  s.cap = p->curve_cap;
  s.stride = std::max(1, p->steps / 64);
  s.sched = p->sched;
  s.lr0 = p->lr0;
  for (int t = 0; t <= p->steps; ++t) {
    s.t = t;
    gen_grad_kernel<<<dim3(unsigned(g.ctas_per_image), unsigned(n)), kGThreads, smem, st>>>(g, d_w, d_b, grad, loss,
                                                                                           d_status);
    gen_adam_kernel<<<unsigned(n), 256, 0, st>>>(g, s, d_w, d_b, d_mask, grad, mom, vel, loss, d_curve, d_status, slots,
                                                 d_grad_w, d_grad_b, d_loss0);
    if (int e = cuda_err("GPU encoder step")) return e;
    if (p->steps == 0) break;
  }
  gen_pad_kernel<<<unsigned(n), 32, 0, st>>>(d_curve, slots, p->curve_cap);  // NaN-pad unused curve slots
  cudaFreeAsync(ws, st);
  return cuda_err("GPU encoder");
}

int rinr_fit_render_general(const int32_t* dims, int nl, int64_t n, const float* d_w, const float* d_b, int32_t h,
                            int32_t w, double omega, int32_t sin_mode, float* d_out, void* stream) {
  GArch A{};
  if (int e = garch_of(dims, nl, A)) return e;
  const GArgs g = make_gargs(A, n, nullptr, h, w, omega, sin_mode == RINR_SIN_ACCURATE);
  const size_t smem = (size_t(A.P + A.PB) + size_t(2) * A.maxw * kTile) * 4;
  if (cudaFuncSetAttribute(gen_render_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return set_error(RINR_ERR_CUDA, "render smem attribute");
  gen_render_kernel<<<dim3(unsigned(g.ctas_per_image), unsigned(n)), kGThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      g, d_w, d_b, d_out);
  return cuda_err("GPU encoder render");
}
