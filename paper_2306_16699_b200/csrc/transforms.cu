// Encoder-side model transforms: magnitude pruning,
// layer-wise affine quantisation and PSNR, one CTA per model (or per
// model x hidden layer / per image).  All weight arithmetic is written with
// explicit IEEE intrinsics (no FMA contraction) so the results are
// bit-identical to the reference's numpy operations.
//
//   prune_l1   compressor.py:100-152
//   quantize   compressor.py:160-202, quantize_codes 205-218
//   psnr       metrics.py:23-41 (u8 path: image.py:49-55)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/rinr_b200_transforms.h"
#include "rinr_internal.h"

namespace rinr {
namespace {

constexpr int kMaxLayers = 64;
constexpr int kThreads = 256;

struct TArch {
  int nl;
  int P;                        // weights per model
  int dims[kMaxLayers + 1];
  int off[kMaxLayers + 1];      // weight offset of matrix l; off[nl] = P
  int boff[kMaxLayers + 1];     // bias offset of layer l
};

__device__ __forceinline__ uint32_t mag_key(float w) {
  // |w| as an order-preserving u32; every NaN collapses to one key so that
  // NaNs rank last and among themselves by position (np.argsort, stable)
  const uint32_t u = __float_as_uint(w) & 0x7fffffffu;
  return u > 0x7f800000u ? 0x7fc00000u : u;
}

// Block-wide sum of one int per thread (all threads must call).
__device__ __forceinline__ int block_sum(int v, int* red) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < (kThreads >> 5); ++i) t += red[i];
  return t;
}

// Block-wide min of one u32 per thread (all threads must call).
__device__ __forceinline__ uint32_t block_min_u32(uint32_t v, int* red) {
  v = __reduce_min_sync(0xffffffffu, v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = int(v);
  __syncthreads();
  uint32_t t = uint32_t(red[0]);
  for (int i = 1; i < (kThreads >> 5); ++i) t = min(t, uint32_t(red[i]));
  return t;
}

// Block-wide exclusive prefix sum over threads in index order.
__device__ __forceinline__ int block_excl_scan(int v, int* red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  __syncthreads();
  if (lane == 31) red[warp] = inc;
  __syncthreads();
  int before = 0;
  for (int i = 0; i < warp; ++i) before += red[i];
  return before + inc - v;
}

// Doom the k smallest keys of [lo, hi) (ties by position) in `dead`:
// T = the smallest key with count(key <= T) >= k, found by bisection over
// the range's key span (finished by a direct select once <= kThreads keys
// remain in the bracket); keys < T are doomed, and of the keys == T the first
// k - count(key < T) in index order.
__device__ void select_smallest(const uint32_t* key, uint8_t* dead, int lo, int hi, int64_t k, int* red,
                                uint32_t* cand) {
  const int tid = threadIdx.x;
  const int len = hi - lo;
  const int per = (len + kThreads - 1) / kThreads;
  const int c0 = lo + tid * per, c1 = min(hi, c0 + per);
  for (int i = c0; i < c1; ++i) dead[i] = 0;
  if (k <= 0) {
    __syncthreads();
    return;
  }
  // T lies between the smallest and the largest key of the range
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  for (int i = c0; i < c1; ++i) {
    kmin = min(kmin, key[i]);
    kmax = max(kmax, key[i]);
  }
  uint32_t a = block_min_u32(kmin, red), b = ~block_min_u32(~kmax, red);
  // invariant: ca = count(key < a) < k <= cb = count(key <= b); bisect until
  // at most one key per thread lies in [a, b], then select among those
  int64_t ca = 0, cb = len;
  while (a < b && cb - ca > kThreads) {
    const uint32_t mid = a + (b - a) / 2;
    int c = 0;
    for (int i = c0; i < c1; ++i) c += key[i] <= mid;
    const int64_t cm = block_sum(c, red);
    if (cm >= k) {
      b = mid;
      cb = cm;
    } else {
      a = mid + 1;
      ca = cm;
    }
  }
  if (a < b) {
    const uint32_t span = b - a;
    int mine = 0;
    for (int i = c0; i < c1; ++i) mine += key[i] - a <= span;
    int pos = block_excl_scan(mine, red);
    for (int i = c0; i < c1; ++i)
      if (key[i] - a <= span) cand[pos++] = key[i];
    __syncthreads();
    const int total = int(cb - ca);
    const uint32_t v = tid < total ? cand[tid] : 0xffffffffu;
    int le = 0;
    for (int q = 0; q < total; ++q) le += cand[q] <= v;
    a = block_min_u32(tid < total && le >= k - ca ? v : 0xffffffffu, red);
  }
  const uint32_t T = a;
  int lt = 0, eq = 0;
  for (int i = c0; i < c1; ++i) {
    lt += key[i] < T;
    eq += key[i] == T;
  }
  const int64_t need = k - block_sum(lt, red);
  // exclusive prefix of tie counts over threads (chunks are in index order)
  __syncthreads();
  red[32 + tid] = eq;
  __syncthreads();
  if (tid == 0) {
    int s = 0;
    for (int i = 0; i < kThreads; ++i) {
      const int v = red[32 + i];
      red[32 + i] = s;
      s += v;
    }
  }
  __syncthreads();
  int64_t rank = red[32 + tid];
  for (int i = c0; i < c1; ++i) {
    const uint32_t u = key[i];
    bool d = u < T;
    if (u == T) {
      d = rank < need;
      ++rank;
    }
    dead[i] = d;
  }
  __syncthreads();
}

__device__ __forceinline__ int64_t k_of(double ratio, int64_t n) {
  // int(math.floor(total_ratio * n + 0.5)) in f64 (compressor.py:124, 143)
  return int64_t(floor(__dadd_rn(__dmul_rn(ratio, double(n)), 0.5)));
}

__global__ void __launch_bounds__(kThreads) prune_kernel(TArch A, float* __restrict__ w, uint8_t* __restrict__ mask,
                                                         const double* __restrict__ ratio, int scope,
                                                         int32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ int red[32 + kThreads];
  __shared__ uint32_t cand[kThreads];
  const int64_t m = blockIdx.x;
  const int P = A.P;
  uint32_t* key = reinterpret_cast<uint32_t*>(sm);
  uint8_t* dead = sm + size_t(P) * 4;
  float* wm = w + m * P;
  uint8_t* mm = mask + m * P;
  const double r = ratio[m];
  if (!(r >= 0.0 && r < 1.0)) {  // compressor.py:117-118
    if (threadIdx.x == 0) status[m] = RINR_ERR_INVALID_INPUT;
    return;
  }
  for (int i = threadIdx.x; i < P; i += kThreads) key[i] = mag_key(wm[i]);
  __syncthreads();
  if (scope == RINR_PRUNE_GLOBAL) {
    select_smallest(key, dead, 0, P, k_of(r, P), red, cand);
  } else {
    for (int l = 0; l < A.nl; ++l)
      select_smallest(key, dead, A.off[l], A.off[l + 1], k_of(r, A.off[l + 1] - A.off[l]), red, cand);
  }
  // new mask = old & ~doomed; no matrix may lose every entry (compressor.py:133-137)
  bool ok = true;
  for (int l = 0; l < A.nl; ++l) {
    int any = 0;
    for (int i = A.off[l] + threadIdx.x; i < A.off[l + 1]; i += kThreads) any |= mm[i] && !dead[i];
    ok = ok && __syncthreads_or(any);
  }
  if (!ok) {
    if (threadIdx.x == 0) status[m] = RINR_ERR_STRUCTURAL;
    return;
  }
  for (int i = threadIdx.x; i < P; i += kThreads) {
    const uint8_t nm = mm[i] && !dead[i];
    mm[i] = nm;
    wm[i] = __fmul_rn(wm[i], nm ? 1.0f : 0.0f);  // np.multiply(w, mask): -0.0 for negative pruned weights
  }
  if (threadIdx.x == 0) status[m] = RINR_OK;
}

__device__ __forceinline__ double block_min_max(double v, bool is_min, double* dred) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, d);
    v = is_min ? fmin(v, o) : fmax(v, o);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) dred[warp] = v;
  __syncthreads();
  double t = dred[0];
  for (int i = 1; i < (kThreads >> 5); ++i) t = is_min ? fmin(t, dred[i]) : fmax(t, dred[i]);
  return t;
}

// grid: n x (nl - 2), one CTA per (model, hidden matrix)
// a / b correctly rounded for b > 0 from y = RN(1/b): q = RN(a y) is within
// one ulp, r = a - b q is exact (FMA), and RN(q + r y) is the correctly rounded
// quotient (Markstein's theorem); quotients here stay in the normal range
// (|a| is a float, b >= 2^-149 / 65535). Zero keeps its sign as in a / b.
__device__ __forceinline__ double div_by_rcp(double a, double b, double y) {
  if (a == 0.0) return a;
  const double q = __dmul_rn(a, y);
  return __fma_rn(__fma_rn(-q, b, a), y, q);
}

__global__ void __launch_bounds__(kThreads) quantize_kernel(TArch A, int bits, float* __restrict__ w,
                                                            const uint8_t* __restrict__ mask,
                                                            const float* __restrict__ bias, double* __restrict__ d_scale,
                                                            int32_t* __restrict__ d_zp, uint8_t* __restrict__ d_const,
                                                            uint16_t* __restrict__ codes, int32_t* __restrict__ status) {
  __shared__ double dred[32];
  __shared__ int ired[32 + kThreads];
  const int NH = A.nl - 2;
  const int64_t m = blockIdx.x / NH;
  const int h = int(blockIdx.x % NH), l = h + 1;
  const int P = A.P, NB = A.boff[A.nl];
  float* wm = w + m * P;
  const uint8_t* mm = mask + m * P;
  // every weight and bias of the model must be finite (compressor.py:172-174)
  int bad = 0;
  for (int i = threadIdx.x; i < P; i += kThreads) bad |= !isfinite(wm[i]);
  for (int i = threadIdx.x; i < NB; i += kThreads) bad |= !isfinite(bias[m * NB + i]);
  if (__syncthreads_or(bad)) {
    if (threadIdx.x == 0 && h == 0) status[m] = RINR_ERR_NUMERIC;
    return;
  }
  const int lo = A.off[l], hi = A.off[l + 1];
  const double qmax = double((1 << bits) - 1);
  // min / max over kept entries (exact in f64; compressor.py:182-186)
  double mn = INFINITY, mx = -INFINITY;
  int kept = 0;
  for (int i = lo + threadIdx.x; i < hi; i += kThreads)
    if (mm[i]) {
      const double v = double(wm[i]);
      mn = fmin(mn, v);
      mx = fmax(mx, v);
      kept = 1;
    }
  const int any = __syncthreads_or(kept);
  mn = block_min_max(mn, true, dred);
  mx = block_min_max(mx, false, dred);
  (void)ired;
  bool constant = !any || mx == mn;
  double scale = 1.0;
  int32_t zp = 0;
  if (!constant) {
    scale = __ddiv_rn(__dsub_rn(mx, mn), qmax);
    const double z = rint(__ddiv_rn(-mn, scale));  // np.round: half to even
    if (!(z >= -2147483648.0 && z < 2147483648.0)) constant = true, scale = 1.0;
    else zp = int32_t(z);
  }
  const int64_t slot = m * NH + h;
  if (threadIdx.x == 0) {
    d_scale[slot] = scale;
    d_zp[slot] = zp;
    d_const[slot] = constant;
  }
  uint16_t* cm = codes + m * P;
  if (constant) {  // values kept exact, no codes (compressor.py:184-186)
    for (int i = lo + threadIdx.x; i < hi; i += kThreads) cm[i] = 0;
    return;
  }
  const double zpd = double(zp), rs = __drcp_rn(scale);
  for (int i = lo + threadIdx.x; i < hi; i += kThreads) {
    // codes = clip(round(w / scale) + zp, 0, qmax); w = f32(scale * (codes - zp)) * mask
    double c = __dadd_rn(rint(div_by_rcp(double(wm[i]), scale, rs)), zpd);
    c = fmin(fmax(c, 0.0), qmax);
    const float q = __double2float_rn(__dmul_rn(scale, __dsub_rn(c, zpd)));
    const float wn = __fmul_rn(q, mm[i] ? 1.0f : 0.0f);
    wm[i] = wn;
    // quantize_codes recomputes from the snapped weights (compressor.py:215-217)
    double c2 = __dadd_rn(rint(div_by_rcp(double(wn), scale, rs)), zpd);
    c2 = fmin(fmax(c2, 0.0), qmax);
    cm[i] = uint16_t(c2);
  }
}

__device__ __forceinline__ double to_unit_u8(float v) {
  // image.as_u8: floor(clip(v, 0, 1) * 255 + 0.5) in f32, then / 255 in f64
  const float c = fminf(fmaxf(v, 0.0f), 1.0f);
  const float u = floorf(__fadd_rn(__fmul_rn(c, 255.0f), 0.5f));
  return __ddiv_rn(double(u), 255.0);
}

__global__ void __launch_bounds__(kThreads) psnr_kernel(const float* __restrict__ a, const float* __restrict__ b,
                                                        int64_t count, int quantized, double* __restrict__ mse,
                                                        double* __restrict__ psnr) {
  __shared__ double dred[32];
  const int64_t m = blockIdx.x;
  const float* pa = a + m * count;
  const float* pb = b + m * count;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += kThreads) {
    const double x = quantized ? to_unit_u8(pa[i]) : double(pa[i]);
    const double y = quantized ? to_unit_u8(pb[i]) : double(pb[i]);
    const double d = __dsub_rn(x, y);
    s = __dadd_rn(s, __dmul_rn(d, d));
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if ((threadIdx.x & 31) == 0) dred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (kThreads >> 5); ++i) t += dred[i];
    const double e = t / double(count);
    mse[m] = e;
    psnr[m] = e == 0.0 ? INFINITY : 10.0 * log10(1.0 / e);
  }
}

// ---- warp-per-model variants (P <= kWarpMaxP): no block barriers ------------

constexpr int kWarpMaxP = 2048;
constexpr int kWarpsPerCta = 8;

// Warp-level select_smallest over [lo, hi) of this warp's keys (same rule).
__device__ void warp_select(const uint32_t* key, uint8_t* dead, int lo, int hi, int64_t k, int lane,
                            uint32_t* cand) {
  const int len = hi - lo;
  const int per = (len + 31) / 32;
  const int c0 = lo + lane * per, c1 = min(hi, c0 + per);
  if (k <= 0) {
    for (int i = c0; i < c1; ++i) dead[i] = 0;
    __syncwarp();
    return;
  }
  uint32_t kmin = 0xffffffffu, kmax = 0u;
  for (int i = c0; i < c1; ++i) {
    kmin = min(kmin, key[i]);
    kmax = max(kmax, key[i]);
  }
  uint32_t a = __reduce_min_sync(0xffffffffu, kmin), b = __reduce_max_sync(0xffffffffu, kmax);
  // invariant: ca = count(key < a) < k <= cb = count(key <= b); bisect until
  // at most 32 keys lie in [a, b], then select among those (as in
  // prune_warp_reg_kernel)
  int ca = 0, cb = len;
  while (a < b && cb - ca > 32) {
    const uint32_t mid = a + (b - a) / 2;
    int c = 0;
    for (int i = c0; i < c1; ++i) c += key[i] <= mid;
    c = int(__reduce_add_sync(0xffffffffu, unsigned(c)));
    if (c >= k) {
      b = mid;
      cb = c;
    } else {
      a = mid + 1;
      ca = c;
    }
  }
  if (a < b) {
    const uint32_t span = b - a;
    int mine = 0;
    for (int i = c0; i < c1; ++i) mine += key[i] - a <= span;
    int incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    int pos = incl - mine;
    for (int i = c0; i < c1; ++i)
      if (key[i] - a <= span) cand[pos++] = key[i];
    __syncwarp();
    const int total = cb - ca;
    const uint32_t v = lane < total ? cand[lane] : 0xffffffffu;
    int le = 0;
    for (int q = 0; q < total; ++q) le += cand[q] <= v;
    a = __reduce_min_sync(0xffffffffu, lane < total && le >= k - ca ? v : 0xffffffffu);
    __syncwarp();
  }
  const uint32_t T = a;
  int lt = 0, eq = 0;
  for (int i = c0; i < c1; ++i) {
    lt += key[i] < T;
    eq += key[i] == T;
  }
  const int64_t need = k - int64_t(__reduce_add_sync(0xffffffffu, unsigned(lt)));
  int incl = eq;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  int64_t rank = incl - eq;
  for (int i = c0; i < c1; ++i) {
    const uint32_t u = key[i];
    bool d = u < T;
    if (u == T) {
      d = rank < need;
      ++rank;
    }
    dead[i] = d;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) prune_warp_kernel(TArch A, int64_t n, float* __restrict__ w,
                                                                      uint8_t* __restrict__ mask,
                                                                      const double* __restrict__ ratio, int scope,
                                                                      int32_t* __restrict__ status) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint32_t sel_cand[kWarpsPerCta][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = int64_t(blockIdx.x) * kWarpsPerCta + warp;
  if (m >= n) return;
  const int P = A.P;
  const int stride = (P * 5 + 15) & ~15;
  uint32_t* key = reinterpret_cast<uint32_t*>(sm + size_t(warp) * stride);
  uint8_t* dead = reinterpret_cast<uint8_t*>(key + P);
  float* wm = w + m * P;
  uint8_t* mm = mask + m * P;
  const double r = ratio[m];
  if (!(r >= 0.0 && r < 1.0)) {
    if (lane == 0) status[m] = RINR_ERR_INVALID_INPUT;
    return;
  }
  for (int i = lane; i < P; i += 32) key[i] = mag_key(wm[i]);
  __syncwarp();
  if (scope == RINR_PRUNE_GLOBAL) {
    warp_select(key, dead, 0, P, k_of(r, P), lane, sel_cand[warp]);
  } else {
    for (int l = 0; l < A.nl; ++l) warp_select(key, dead, A.off[l], A.off[l + 1], k_of(r, A.off[l + 1] - A.off[l]), lane,
                                              sel_cand[warp]);
  }
  bool ok = true;
  for (int l = 0; l < A.nl; ++l) {
    int any = 0;
    for (int i = A.off[l] + lane; i < A.off[l + 1]; i += 32) any |= mm[i] && !dead[i];
    ok = ok && __any_sync(0xffffffffu, any);
  }
  if (!ok) {
    if (lane == 0) status[m] = RINR_ERR_STRUCTURAL;
    return;
  }
  for (int i = lane; i < P; i += 32) {
    const uint8_t nm = mm[i] && !dead[i];
    mm[i] = nm;
    wm[i] = __fmul_rn(wm[i], nm ? 1.0f : 0.0f);
  }
  if (lane == 0) status[m] = RINR_OK;
}

// Global-scope prune of one small model (P <= 32 KPL) per warp with the keys
// in registers, interleaved (key j of a lane is entry 32 j + lane, so global
// loads and stores are coalesced): the same bisection for T, with per-lane
// counts and one REDUX per step, then ties ranked in index order by ballots.
// CTAs per SM: the most that fit each key count without spills (old mask
// and doomed bits are packed into one word per lane).
template <int KPL>
constexpr int prune_reg_ctas() { return KPL >= 16 ? 4 : (KPL >= 10 ? 5 : 6); }

template <int KPL>
__global__ void __launch_bounds__(kWarpsPerCta * 32, prune_reg_ctas<KPL>())
    prune_warp_reg_kernel(TArch A, int64_t n, float* __restrict__ w, uint8_t* __restrict__ mask,
                          const double* __restrict__ ratio, int32_t* __restrict__ status) {
  __shared__ uint32_t sel_cand[kWarpsPerCta][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = int64_t(blockIdx.x) * kWarpsPerCta + warp;
  if (m >= n) return;
  const int P = A.P;
  float* wm = w + m * P;
  uint8_t* mm = mask + m * P;
  const double r = ratio[m];
  if (!(r >= 0.0 && r < 1.0)) {
    if (lane == 0) status[m] = RINR_ERR_INVALID_INPUT;
    return;
  }
  uint32_t key[KPL];
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const int i = 32 * j + lane;
    key[j] = i < P ? mag_key(wm[i]) : 0xffffffffu;  // padding ranks after every real key
  }
  const int k = int(k_of(r, P));  // P <= 512
  uint32_t dead = 0;  // bit j: entry 32 j + lane is pruned
  if (k > 0) {
    // T lies between the smallest and the largest real key
    uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll
    for (int j = 0; j < KPL; ++j)
      if (32 * j + lane < P) {
        lo = min(lo, key[j]);
        hi = max(hi, key[j]);
      }
    uint32_t a = __reduce_min_sync(0xffffffffu, lo), b = __reduce_max_sync(0xffffffffu, hi);
    // invariant: ca = count(key < a) < k <= cb = count(key <= b); bisect
    // until at most 32 keys lie in [a, b], then select among those directly
    int ca = 0, cb = P;
    while (a < b && cb - ca > 32) {
      const uint32_t mid = a + (b - a) / 2;
      int c = 0;
#pragma unroll
      for (int j = 0; j < KPL; ++j) c += key[j] <= mid;
      c = int(__reduce_add_sync(0xffffffffu, unsigned(c)));
      if (c >= k) {
        b = mid;
        cb = c;
      } else {
        a = mid + 1;
        ca = c;
      }
    }
    if (a < b) {
      // compact the <= 32 keys of [a, b] (padding keys are above b) into one
      // slot per lane, then T = the smallest candidate with
      // count(candidates <= T) >= k - ca
      uint32_t* cand = sel_cand[warp];
      const uint32_t below = (1u << lane) - 1u, span = b - a;
      int base = 0;
#pragma unroll
      for (int j = 0; j < KPL; ++j) {
        const bool in = key[j] - a <= span;
        const uint32_t bal = __ballot_sync(0xffffffffu, in);
        if (in) cand[base + __popc(bal & below)] = key[j];
        base += __popc(bal);
      }
      __syncwarp();
      const uint32_t mine = lane < base ? cand[lane] : 0xffffffffu;
      int le = 0;
      for (int q = 0; q < base; ++q) le += cand[q] <= mine;
      a = __reduce_min_sync(0xffffffffu, lane < base && le >= k - ca ? mine : 0xffffffffu);
      __syncwarp();
    }
    const uint32_t T = a;
    int lt = 0;
#pragma unroll
    for (int j = 0; j < KPL; ++j) lt += key[j] < T;
    const int need = k - int(__reduce_add_sync(0xffffffffu, unsigned(lt)));
    const uint32_t below = (1u << lane) - 1u;
    int base = 0;  // ties in earlier rows
#pragma unroll
    for (int j = 0; j < KPL; ++j) {
      const uint32_t eq = __ballot_sync(0xffffffffu, key[j] == T);
      const bool d = key[j] < T || (key[j] == T && base + __popc(eq & below) < need);
      dead |= uint32_t(d) << j;
      base += __popc(eq);
    }
  }
  // structural check: every matrix keeps an entry (layers are index ranges)
  uint32_t keep = 0;  // bit j: entry 32 j + lane stays (old mask and not doomed)
  uint32_t surv = 0;  // bit l: this lane keeps an entry of matrix l
  int l = 0;
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const int i = 32 * j + lane;
    if (i < P) {
      const bool kp = mm[i] && !((dead >> j) & 1u);
      keep |= uint32_t(kp) << j;
      while (i >= A.off[l + 1]) ++l;
      if (kp) surv |= 1u << l;
    }
  }
  surv = __reduce_or_sync(0xffffffffu, surv);
  if (surv != (1u << A.nl) - 1u) {
    if (lane == 0) status[m] = RINR_ERR_STRUCTURAL;
    return;
  }
#pragma unroll
  for (int j = 0; j < KPL; ++j) {
    const int i = 32 * j + lane;
    if (i < P) {
      const uint8_t nm = (keep >> j) & 1u;
      mm[i] = nm;
      wm[i] = __fmul_rn(wm[i], nm ? 1.0f : 0.0f);
    }
  }
  if (lane == 0) status[m] = RINR_OK;
}

__device__ __forceinline__ double warp_min_max(double v, bool is_min) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const double o = __shfl_xor_sync(0xffffffffu, v, d);
    v = is_min ? fmin(v, o) : fmax(v, o);
  }
  return v;
}

__global__ void __launch_bounds__(kWarpsPerCta * 32) quantize_warp_kernel(
    TArch A, int64_t n, int bits, float* __restrict__ w, const uint8_t* __restrict__ mask,
    const float* __restrict__ bias, double* __restrict__ d_scale, int32_t* __restrict__ d_zp,
    uint8_t* __restrict__ d_const, uint16_t* __restrict__ codes, int32_t* __restrict__ status) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = int64_t(blockIdx.x) * kWarpsPerCta + warp;
  if (m >= n) return;
  const int NH = A.nl - 2;
  const int P = A.P, NB = A.boff[A.nl];
  float* wm = w + m * P;
  const uint8_t* mm = mask + m * P;
  uint16_t* cm = codes + m * P;
  int bad = 0;
  for (int i = lane; i < P; i += 32) bad |= !isfinite(wm[i]);
  for (int i = lane; i < NB; i += 32) bad |= !isfinite(bias[m * NB + i]);
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) status[m] = RINR_ERR_NUMERIC;
    return;
  }
  const double qmax = double((1 << bits) - 1);
  for (int h = 0; h < NH; ++h) {
    const int lo = A.off[h + 1], hi = A.off[h + 2];
    double mn = INFINITY, mx = -INFINITY;
    int kept = 0;
    for (int i = lo + lane; i < hi; i += 32)
      if (mm[i]) {
        const double v = double(wm[i]);
        mn = fmin(mn, v);
        mx = fmax(mx, v);
        kept = 1;
      }
    const bool any = __any_sync(0xffffffffu, kept);
    mn = warp_min_max(mn, true);
    mx = warp_min_max(mx, false);
    bool constant = !any || mx == mn;
    double scale = 1.0;
    int32_t zp = 0;
    if (!constant) {
      scale = __ddiv_rn(__dsub_rn(mx, mn), qmax);
      const double z = rint(__ddiv_rn(-mn, scale));
      if (!(z >= -2147483648.0 && z < 2147483648.0)) constant = true, scale = 1.0;
      else zp = int32_t(z);
    }
    if (lane == 0) {
      d_scale[m * NH + h] = scale;
      d_zp[m * NH + h] = zp;
      d_const[m * NH + h] = constant;
    }
    if (constant) {
      for (int i = lo + lane; i < hi; i += 32) cm[i] = 0;
      continue;
    }
    const double zpd = double(zp), rs = __drcp_rn(scale);
    for (int i = lo + lane; i < hi; i += 32) {
      double c = __dadd_rn(rint(div_by_rcp(double(wm[i]), scale, rs)), zpd);
      c = fmin(fmax(c, 0.0), qmax);
      const float q = __double2float_rn(__dmul_rn(scale, __dsub_rn(c, zpd)));
      const float wn = __fmul_rn(q, mm[i] ? 1.0f : 0.0f);
      wm[i] = wn;
      double c2 = __dadd_rn(rint(div_by_rcp(double(wn), scale, rs)), zpd);
      c2 = fmin(fmax(c2, 0.0), qmax);
      cm[i] = uint16_t(c2);
    }
  }
}

int arch_of(const int32_t* dims, int nl, TArch& A) {
  if (!dims || nl < 1 || nl > kMaxLayers) return set_error(RINR_ERR_INVALID_INPUT, "bad architecture");
  A.nl = nl;
  int64_t p = 0, q = 0;
  for (int l = 0; l <= nl; ++l) {
    if (dims[l] < 1) return set_error(RINR_ERR_INVALID_INPUT, "architecture dims must be >= 1");
    A.dims[l] = dims[l];
  }
  for (int l = 0; l < nl; ++l) {
    A.off[l] = int(p);
    A.boff[l] = int(q);
    p += int64_t(dims[l]) * dims[l + 1];
    q += dims[l + 1];
  }
  if (p > (1 << 24)) return set_error(RINR_ERR_UNSUPPORTED, "model too large for the transform kernels");
  A.off[nl] = int(p);
  A.boff[nl] = int(q);
  A.P = int(p);
  return RINR_OK;
}

int cuda_check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(RINR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return RINR_OK;
}

}  // namespace
}  // namespace rinr

using namespace rinr;

extern "C" int rinr_prune_l1(const int32_t* dims, int nl, int64_t n, float* d_w, uint8_t* d_mask,
                             const double* d_ratio, int scope, int32_t* d_status, void* stream) {
  clear_error();
  TArch A;
  if (int e = arch_of(dims, nl, A)) return e;
  if (n < 0 || (n > 0 && (!d_w || !d_mask || !d_ratio || !d_status)))
    return set_error(RINR_ERR_INVALID_INPUT, "null buffer or negative n");
  if (scope != RINR_PRUNE_GLOBAL && scope != RINR_PRUNE_PER_LAYER)
    return set_error(RINR_ERR_INVALID_INPUT, "unknown prune scope");
  if (n == 0) return RINR_OK;
  if (scope == RINR_PRUNE_GLOBAL && A.P <= 512 && A.nl <= 31) {  // keys in registers, one warp per model
    const unsigned grid = unsigned((n + kWarpsPerCta - 1) / kWarpsPerCta);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
#define RINR_PRUNE_REG(K) prune_warp_reg_kernel<K><<<grid, kWarpsPerCta * 32, 0, st>>>(A, n, d_w, d_mask, d_ratio, d_status)
    if (A.P <= 128) RINR_PRUNE_REG(4);
    else if (A.P <= 256) RINR_PRUNE_REG(8);
    else if (A.P <= 320) RINR_PRUNE_REG(10);
    else if (A.P <= 384) RINR_PRUNE_REG(12);
    else RINR_PRUNE_REG(16);
#undef RINR_PRUNE_REG
    return cuda_check("prune_l1 launch");
  }
  if (A.P <= kWarpMaxP) {  // small models: one warp each
    const size_t smem = size_t(kWarpsPerCta) * ((A.P * 5 + 15) & ~15);
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(prune_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
      return cuda_check("prune_l1 smem attribute");
    prune_warp_kernel<<<unsigned((n + kWarpsPerCta - 1) / kWarpsPerCta), kWarpsPerCta * 32, smem,
                        static_cast<cudaStream_t>(stream)>>>(A, n, d_w, d_mask, d_ratio, scope, d_status);
    return cuda_check("prune_l1 launch");
  }
  const size_t smem = size_t(A.P) * 5;
  if (smem > 200 * 1024) return set_error(RINR_ERR_UNSUPPORTED, "model too large for prune_l1 on one CTA");
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(prune_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
    return cuda_check("prune_l1 smem attribute");
  prune_kernel<<<unsigned(n), kThreads, smem, static_cast<cudaStream_t>(stream)>>>(A, d_w, d_mask, d_ratio, scope,
                                                                                    d_status);
  return cuda_check("prune_l1 launch");
}

extern "C" int rinr_quantize(const int32_t* dims, int nl, int64_t n, int bits, float* d_w, const uint8_t* d_mask,
                             const float* d_b, double* d_scale, int32_t* d_zp, uint8_t* d_const, uint16_t* d_codes,
                             int32_t* d_status, void* stream) {
  clear_error();
  TArch A;
  if (int e = arch_of(dims, nl, A)) return e;
  if (bits != 8 && bits != 16) return set_error(RINR_ERR_INVALID_INPUT, "bits must be 8 or 16");
  if (n < 0) return set_error(RINR_ERR_INVALID_INPUT, "negative n");
  if (nl < 3 || n == 0) return RINR_OK;  // no hidden matrices
  if (!d_w || !d_mask || !d_b || !d_scale || !d_zp || !d_const || !d_codes || !d_status)
    return set_error(RINR_ERR_INVALID_INPUT, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(d_status, 0, size_t(n) * sizeof(int32_t), st) != cudaSuccess) return cuda_check("status reset");
  if (A.P <= kWarpMaxP)
    quantize_warp_kernel<<<unsigned((n + kWarpsPerCta - 1) / kWarpsPerCta), kWarpsPerCta * 32, 0, st>>>(
        A, n, bits, d_w, d_mask, d_b, d_scale, d_zp, d_const, d_codes, d_status);
  else
    quantize_kernel<<<unsigned(n * (nl - 2)), kThreads, 0, st>>>(A, bits, d_w, d_mask, d_b, d_scale, d_zp, d_const,
                                                                 d_codes, d_status);
  return cuda_check("quantize launch");
}

extern "C" int rinr_psnr(const float* d_a, const float* d_b, int64_t n, int64_t count, int quantized, double* d_mse,
                         double* d_psnr, void* stream) {
  clear_error();
  if (n < 0 || count < 1) return set_error(RINR_ERR_INVALID_INPUT, "need n >= 0 images of count >= 1 values");
  if (n == 0) return RINR_OK;
  if (!d_a || !d_b || !d_mse || !d_psnr) return set_error(RINR_ERR_INVALID_INPUT, "null buffer");
  psnr_kernel<<<unsigned(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(d_a, d_b, count, quantized, d_mse,
                                                                               d_psnr);
  return cuda_check("psnr launch");
}
