// Batched SIREN fitting: encoder._train
// (encoder.py:66-85) = full-batch Adam (net.py:268-300) over
// net.loss_and_grad (net.py:217-265), one CTA per image, every step of a
// round inside one launch.
//
// Architecture (2, H, H, 3), 8 <= H <= 16, omega from the record.  Per step:
//   1. forward + backward of every pixel, the loss accumulated in f64
//      (resid.astype(f64)**2), and the gradient sums over pixels:
//        * MUFU sine, H < 16 (mma_pass): register-resident mma.sync bf16
//          3-pass chains in fragment layout, gradient sums accumulated in MMA
//          registers through movmatrix transposes; 2 CTAs per SM;
//        * accurate sine or H = 16 (pixel_pass): fp32 FFMA, one thread per
//          pixel pair, rows staged in shared memory and reduced by 3xTF32
//          mma.m16n8k8 (tc_reduce) or a lane-tiled FFMA loop (H = 16);
//   2. cross-warp sums in shared memory, then the Adam update in numpy's f32
//      operation order, with the mask re-applied.
// Shared memory holds the weights (compute copy, padded rows, plus a
// transposed W1), Adam moments, masks, per-warp partial gradients and either
// the staging tiles (FFMA pass, ~180 KB) or the per-warp B fragments and
// coordinate tables (MMA pass, ~42 KB).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "../../include/rinr_b200_encoder.h"
#include "device_common.cuh"
#include "mma_chain.cuh"
#include "rinr_internal.h"

namespace rinr {
namespace {

#ifndef RINR_FIT_NPX
#define RINR_FIT_NPX 2  // pixels per thread
#endif
constexpr int kFitWarps = 16;
constexpr int kFitThreads = kFitWarps * 32;
constexpr int kFragGroups = 6;  // uint4 B-fragment groups per lane (MMA pass)
constexpr int kPixTable = 2048;  // MMA pass: per-pixel coordinate / target tables up to this many pixels
constexpr int kStage = 76;  // floats per staged pixel (stride 76: conflict-free STS.128)
// staged pixel: a0 [0,16) a1 [16,32) d1 [32,48) d0 [48,64) d2 [64,68) (x, y) [68,70)
constexpr int SA0 = 0, SA1 = 16, SD1 = 32, SD0 = 48, SD2 = 64, SXY = 68;

template <int H>
struct FitLayout {
  // canonical parameter order = transform layout: W0 [H][2], W1 [H][H], W2 [3][H] | b0, b1, b2
  static constexpr int P = 2 * H + H * H + 3 * H;
  static constexpr int PB = 2 * H + 3;
  static constexpr int NPAR = P + PB;
  static constexpr int NPAR_PAD = (NPAR + 3) & ~3;
  // shared compute copy (padded rows)
  // W1TS: a transposed copy of W1 (column k at W1TS + 16k), so layer 1 runs
  // k-outer with H independent accumulators per pixel instead of H-long chains
  static constexpr int W0S = 0, W1S = 32, W2S = 32 + 256, B0S = W2S + 64, B1S = B0S + 16, B2S = B1S + 16;
  static constexpr int W1TS = B2S + 16;
  static constexpr int WS = W1TS + 256;
  __device__ static int slot(int p) {
    if (p < 2 * H) return W0S + p;  // row o = p/2 of 2 floats
    p -= 2 * H;
    if (p < H * H) return W1S + (p / H) * 16 + p % H;
    p -= H * H;
    if (p < 3 * H) return W2S + (p / H) * 16 + p % H;
    p -= 3 * H;
    if (p < H) return B0S + p;
    p -= H;
    if (p < H) return B1S + p;
    return B2S + (p - H);
  }
  // store parameter p (canonical order) into the compute copy, W1 twice
  __device__ static void put(float* ws, int p, float v) {
    ws[slot(p)] = v;
    const int q = p - 2 * H;
    if (q >= 0 && q < H * H) ws[W1TS + (q % H) * 16 + q / H] = v;
  }
  // fixed part; the MMA pass adds no staging tiles but (h + w) coordinate floats
  static constexpr size_t smem_bytes(int npx, bool stage = true) {
    return sizeof(float) * (size_t(WS) + 2 * NPAR_PAD + ((P + 3) & ~3) + size_t(kFitWarps / npx) * NPAR_PAD +
                            (stage ? size_t(kFitWarps / npx) * 32 * npx * kStage : 0)) +
           sizeof(double) * kFitWarps + (stage ? 0 : sizeof(uint32_t) * 4 * 32 * kFragGroups * (kFitWarps / npx));
  }
};

struct FitArgs {
  int64_t n;
  float* w;
  float* b;
  const uint8_t* mask;
  const float* images;
  int h, wd, hw, steps, cap;
  double inv_wm1, inv_hm1;
  double lr0, omega;
  double* curve;
  int32_t* status;
  float* grad_w;
  float* grad_b;
  double* loss0;
  const float* sched;  // [steps][3] (lr, c1, c2) or null
};

template <bool ACC>
__device__ __forceinline__ void sincos_(float u, float& s, float& c) {
  if constexpr (ACC) sincosf(u, &s, &c);
  else __sincosf(u, &s, &c);
}

// Weights are read with volatile vector loads: ptxas may neither hoist nor
// merge them, so the ~300 loop-invariant weights are re-read per pixel (one
// LDS.128 per 4 weights, broadcast) instead of being pinned in registers
// across the pixel loop, which would spill.
__device__ __forceinline__ float4 wld4(const float* p) {
  float4 v;
  asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

template <int H>
__device__ __forceinline__ void wrow(const float* p, float (&r)[16]) {
#pragma unroll
  for (int k = 0; k < 16; k += 4) {
    if (k < H) {
      const float4 v = wld4(p + k);
      r[k] = v.x;
      r[k + 1] = v.y;
      r[k + 2] = v.z;
      r[k + 3] = v.w;
    }
  }
}

// Forward (+ backward when BWD) of NPX pixels per thread: a0/c0/a1/c1
// (c = omega cos(omega z)); on return of the backward, c1 holds d1 and c0
// holds d0.  Every weight row loaded from shared memory serves all NPX pixels.
template <int H, bool ACC, bool BWD, int NPX>
__device__ __forceinline__ void pixel_pass(const float* __restrict__ ws, const float (&x)[NPX], const float (&y)[NPX],
                                           const float (&tg)[NPX][3], float om, float s2, float (&a0)[NPX][16],
                                           float (&c0)[NPX][16], float (&a1)[NPX][16], float (&c1)[NPX][16],
                                           float (&d2)[NPX][3], float (&out)[NPX][3], double (&lp)[NPX]) {
  using L = FitLayout<H>;
  float r[16], bb[16];
  // layer 0: 2 -> H (W0 rows are float2 pairs: 8 rows per 4 loads)
  wrow<H>(ws + L::B0S, bb);
#pragma unroll
  for (int o0 = 0; o0 < H; o0 += 2) {
    const float4 w = wld4(ws + L::W0S + 2 * o0);  // rows o0, o0+1
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int o = o0 + h;
      if (o < H) {
        const float wx = h ? w.z : w.x, wy = h ? w.w : w.y;
#pragma unroll
        for (int p = 0; p < NPX; ++p) {
          const float z = __fadd_rn(fmaf(y[p], wy, __fmul_rn(x[p], wx)), bb[o]);
          float s, c;
          sincos_<ACC>(__fmul_rn(om, z), s, c);
          a0[p][o] = s;
          c0[p][o] = __fmul_rn(om, c);
        }
      }
    }
  }
  // layer 1: H -> H, k-outer over W1's columns: NPX*H independent FMA
  // chains, each summing k = 0..H-1 in order (the same rounding as a dot loop)
#pragma unroll
  for (int p = 0; p < NPX; ++p)
#pragma unroll
    for (int o = 0; o < 16; ++o) a1[p][o] = 0.0f;
#pragma unroll
  for (int k = 0; k < H; ++k) {
    wrow<H>(ws + L::W1TS + 16 * k, r);
#pragma unroll
    for (int p = 0; p < NPX; ++p)
#pragma unroll
      for (int o = 0; o < H; ++o) a1[p][o] = fmaf(a0[p][k], r[o], a1[p][o]);
  }
  wrow<H>(ws + L::B1S, bb);
#pragma unroll
  for (int o = 0; o < H; ++o) {
#pragma unroll
    for (int p = 0; p < NPX; ++p) {
      float s, c;
      sincos_<ACC>(__fmul_rn(om, __fadd_rn(a1[p][o], bb[o])), s, c);
      a1[p][o] = s;
      c1[p][o] = __fmul_rn(om, c);
    }
  }
  // layer 2: H -> 3 (affine)
  const float4 b2 = wld4(ws + L::B2S);
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    wrow<H>(ws + L::W2S + 16 * j, r);
#pragma unroll
    for (int p = 0; p < NPX; ++p) {
      float acc = 0.0f;
#pragma unroll
      for (int k = 0; k < H; ++k) acc = fmaf(a1[p][k], r[k], acc);
      out[p][j] = __fadd_rn(acc, j == 0 ? b2.x : (j == 1 ? b2.y : b2.z));
    }
  }
  if constexpr (BWD) {
#pragma unroll
    for (int p = 0; p < NPX; ++p)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float e = __fsub_rn(out[p][j], tg[p][j]);
        lp[p] += double(e) * double(e);
        d2[p][j] = __fmul_rn(s2, e);  // (2.0 * scale) * resid
      }
    // d1 = (d2 @ W2) * c1
    float g[NPX][16];
    wrow<H>(ws + L::W2S, r);
#pragma unroll
    for (int p = 0; p < NPX; ++p)
#pragma unroll
      for (int k = 0; k < H; ++k) g[p][k] = __fmul_rn(d2[p][0], r[k]);
#pragma unroll
    for (int j = 1; j < 3; ++j) {
      wrow<H>(ws + L::W2S + 16 * j, r);
#pragma unroll
      for (int p = 0; p < NPX; ++p)
#pragma unroll
        for (int k = 0; k < H; ++k) g[p][k] = fmaf(d2[p][j], r[k], g[p][k]);
    }
#pragma unroll
    for (int p = 0; p < NPX; ++p)
#pragma unroll
      for (int k = 0; k < H; ++k) c1[p][k] = __fmul_rn(g[p][k], c1[p][k]);
    // d0 = (d1 @ W1) * c0, row-outer so each W1 row is 4 vector loads
#pragma unroll
    for (int p = 0; p < NPX; ++p)
#pragma unroll
      for (int k = 0; k < H; ++k) g[p][k] = 0.0f;
#pragma unroll
    for (int o = 0; o < H; ++o) {
      wrow<H>(ws + L::W1S + 16 * o, r);
#pragma unroll
      for (int p = 0; p < NPX; ++p)
#pragma unroll
        for (int k = 0; k < H; ++k) g[p][k] = fmaf(c1[p][o], r[k], g[p][k]);
    }
#pragma unroll
    for (int p = 0; p < NPX; ++p)
#pragma unroll
      for (int k = 0; k < H; ++k) c0[p][k] = __fmul_rn(g[p][k], c0[p][k]);
  }
}

// mma.sync m16n8k8 tf32 (f32 accumulate).  Operands are f32 registers; the
// tensor core reads their top 19 bits.
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// x = hi + lo with hi = x's tf32 value (what the tensor core reads) and lo
// the exact remainder (itself read as tf32): 3-pass products are fp32-accurate.
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  const uint32_t u = __float_as_uint(x);
  hi = u;
  lo = __float_as_uint(__fsub_rn(x, __uint_as_float(u & 0xffffe000u)));
}

// Outer-product gradient sums of one staged chunk on tensor cores (H < 16):
//   gW1 | gb1 = d1^T [a0 | 1],   (gW2 | gb2)^T = [a1 | 1]^T d2,   gW0 | gb0 = d0^T [x y 1]
// (gW2 is computed transposed so its 3 rows fill one N = 8 tile instead of
// padding M = 16 over two tiles: 12 MMAs per 8 pixels instead of 15)
// as M16 x N x K(=pixels) GEMMs in 3xTF32 (hi*hi + hi*lo + lo*hi), then the
// fragments are added to the warp's partial row (each entry has one owner lane).
template <int H>
__device__ __forceinline__ void tc_reduce(const float* st, int rows, float* pw, int lane) {
  using L = FitLayout<H>;
  const int g = lane >> 2, tq = lane & 3;
  // one accumulator per 3xTF32 pass: 15 independent MMA chains per k-step
  float c1[3][2][4] = {}, c2[3][4] = {}, c0[3][4] = {};
  for (int kb = 0; kb < rows; kb += 8) {
    const float* r0 = st + (kb + tq) * kStage;      // pixel kb + tq
    const float* r1 = st + (kb + tq + 4) * kStage;  // pixel kb + tq + 4
    // A operands (rows = unit, K = pixel): d1^T, d0^T; d2 is a B operand (N = j)
    uint32_t a1h[4], a1l[4], a0h[4], a0l[4], d2h[2], d2l[2];
    tf32_split(r0[SD1 + g], a1h[0], a1l[0]);
    tf32_split(r0[SD1 + g + 8], a1h[1], a1l[1]);
    tf32_split(r1[SD1 + g], a1h[2], a1l[2]);
    tf32_split(r1[SD1 + g + 8], a1h[3], a1l[3]);
    tf32_split(r0[SD0 + g], a0h[0], a0l[0]);
    tf32_split(r0[SD0 + g + 8], a0h[1], a0l[1]);
    tf32_split(r1[SD0 + g], a0h[2], a0l[2]);
    tf32_split(r1[SD0 + g + 8], a0h[3], a0l[3]);
    tf32_split(g < 3 ? r0[SD2 + (g & 3)] : 0.0f, d2h[0], d2l[0]);
    tf32_split(g < 3 ? r1[SD2 + (g & 3)] : 0.0f, d2h[1], d2l[1]);
    uint32_t b1h[2][2], b1l[2][2], b2h[2][2], b2l[2][2], b0h[2], b0l[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      tf32_split(r0[SA0 + 8 * j + g], b1h[j][0], b1l[j][0]);  // B = [a0 | 1]
      tf32_split(r1[SA0 + 8 * j + g], b1h[j][1], b1l[j][1]);
      tf32_split(r0[SA1 + 8 * j + g], b2h[j][0], b2l[j][0]);  // [a1 | 1] (gW2^T A operand)
      tf32_split(r1[SA1 + 8 * j + g], b2h[j][1], b2l[j][1]);
    }
    tf32_split(g < 4 ? r0[SXY + (g & 3)] : 0.0f, b0h[0], b0l[0]);  // B = [x y 1 0 ...]
    tf32_split(g < 4 ? r1[SXY + (g & 3)] : 0.0f, b0h[1], b0l[1]);
    // A = [a1 | 1]^T: the B values loaded for gW2 before, regrouped
    const uint32_t e2h[4] = {b2h[0][0], b2h[1][0], b2h[0][1], b2h[1][1]};
    const uint32_t e2l[4] = {b2l[0][0], b2l[1][0], b2l[0][1], b2l[1][1]};
#pragma unroll
    for (int j = 0; j < 2; ++j) mma_tf32(c1[0][j], a1h, b1h[j][0], b1h[j][1]);
    mma_tf32(c2[0], e2h, d2h[0], d2h[1]);
    mma_tf32(c0[0], a0h, b0h[0], b0h[1]);
#pragma unroll
    for (int j = 0; j < 2; ++j) mma_tf32(c1[1][j], a1h, b1l[j][0], b1l[j][1]);
    mma_tf32(c2[1], e2h, d2l[0], d2l[1]);
    mma_tf32(c0[1], a0h, b0l[0], b0l[1]);
#pragma unroll
    for (int j = 0; j < 2; ++j) mma_tf32(c1[2][j], a1l, b1h[j][0], b1h[j][1]);
    mma_tf32(c2[2], e2l, d2h[0], d2h[1]);
    mma_tf32(c0[2], a0l, b0h[0], b0h[1]);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
#pragma unroll
    for (int j = 0; j < 2; ++j) c1[0][j][e] = __fadd_rn(c1[0][j][e], __fadd_rn(c1[1][j][e], c1[2][j][e]));
    c2[0][e] = __fadd_rn(c2[0][e], __fadd_rn(c2[1][e], c2[2][e]));
    c0[0][e] = __fadd_rn(c0[0][e], __fadd_rn(c0[1][e], c0[2][e]));
  }
  // C fragment: c[0] (row g, col 2tq), c[1] (g, 2tq+1), c[2] (g+8, 2tq), c[3] (g+8, 2tq+1)
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int row = g + 8 * (e >> 1), colb = 2 * tq + (e & 1);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = 8 * j + colb;
      if (row < H) {  // gW1[o][k] and gb1[o] (ones column k == H)
        if (col < H) pw[2 * H + row * H + col] += c1[0][j][e];
        else if (col == H) pw[L::P + H + row] += c1[0][j][e];
      }
    }
    if (colb < 3) {  // transposed: row = unit k of a1 (k == H: gb2), col = output j
      if (row < H) pw[2 * H + H * H + colb * H + row] += c2[0][e];
      else if (row == H) pw[L::P + 2 * H + colb] += c2[0][e];
    }
    if (row < H) {  // gW0[o][0..1] and gb0[o]
      if (colb < 2) pw[2 * row + colb] += c0[0][e];
      else if (colb == 2) pw[L::P + row] += c0[0][e];
    }
  }
}

// ---------------------------------------------------------------------------
// Tensor-core pixel pass (MUFU sine mode, H < 16): pixel_pass's per-pixel
// network as register-resident mma.sync.m16n8k16 chains, like the decoder's
// (mma_chain.cuh).  A warp evaluates 16-pixel m-tiles; the f32 accumulator
// fragment of n-tiles 0 / 1 is the A fragment of the next product, so
//   z1 = a0 W1^T + b1,  out = a1 W2^T + b2,  d1 = (d2 W2) * c1,  d0 = (d1 W1) * c0
// never leave registers.  Products are bf16 3-pass (Ah*Bh + Al*Bh + Ah*Bl,
// round-to-nearest split: about 2^-17 relative per product), inside the MUFU mode's
// stated gradient tolerance; the accurate-sine mode keeps the fp32 FFMA pass.
// Layer 0 (K = 2) is FFMA in the same fragment layout.  C-fragment element e
// of n-tile j: pixel row g + 8(e >> 1), unit 8j + 2tq + (e & 1).
// ---------------------------------------------------------------------------
// B fragments live in a per-warp shared block (6 uint4 groups x 32 lanes,
// read with one LDS.128 right before each use, keeping ~24 registers free):
//   group 0/1: forward W1 n-tile 0/1, B[k][n] = W1[n][k], {b0 hi, b1 hi, b0 lo, b1 lo}
//   group 2/3: backward W1 n-tile 0/1, B[o][k] = W1[o][k]
//   group 4:   forward W2, B[k][j] = W2[j][k] (3 valid columns)
//   group 5:   backward W2 n-tiles 0/1, B[j][o] = W2[j][o] (K = 3 valid): {hi0, lo0, hi1, lo1}
struct FitFrags {
  float w0x[2][2], w0y[2][2], b0[2][2], b1[2][2], b2[2];  // this lane's units / outputs
};

__device__ __forceinline__ uint4 frag_ld(const uint4* p) {
  uint4 v;
  asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

template <int H>
// Every fragment carries omega: forward z' = omega z goes straight into the
// sine, and the backward products (d W) omega times cos(z') are the reference's
// (d W) * (omega cos(omega z)).
__device__ __forceinline__ void load_frags(const float* ws, int lane, float om, FitFrags& F, uint4* fq) {
  using L = FitLayout<H>;
  const int g = lane >> 2, tq = lane & 3;
  // W1 rows are zero padded to 16 x 16, W2 to 4 x 16 (ws is zeroed at start)
  auto W1 = [&](int o, int k) { return ws[L::W1S + 16 * o + k]; };
  auto W2 = [&](int j, int k) { return j < 3 ? ws[L::W2S + 16 * j + k] : 0.0f; };
  uint32_t w2b[4];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int n = 8 * j + g;
    uint32_t f[4], b[4];
    pack_act<true>(om * W1(n, 2 * tq), om * W1(n, 2 * tq + 1), f[0], f[2]);
    pack_act<true>(om * W1(n, 2 * tq + 8), om * W1(n, 2 * tq + 9), f[1], f[3]);
    pack_act<true>(om * W1(2 * tq, n), om * W1(2 * tq + 1, n), b[0], b[2]);
    pack_act<true>(om * W1(2 * tq + 8, n), om * W1(2 * tq + 9, n), b[1], b[3]);
    pack_act<true>(om * W2(2 * tq, n), om * W2(2 * tq + 1, n), w2b[2 * j], w2b[2 * j + 1]);
    fq[32 * j] = make_uint4(f[0], f[1], f[2], f[3]);
    fq[32 * (2 + j)] = make_uint4(b[0], b[1], b[2], b[3]);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int u = 8 * j + 2 * tq + e;
      F.w0x[j][e] = om * ws[L::W0S + 2 * u];
      F.w0y[j][e] = om * ws[L::W0S + 2 * u + 1];
      F.b0[j][e] = om * ws[L::B0S + u];
      F.b1[j][e] = om * ws[L::B1S + u];
    }
  }
  uint32_t f[4];
  pack_act<true>(W2(g, 2 * tq), W2(g, 2 * tq + 1), f[0], f[2]);
  pack_act<true>(W2(g, 2 * tq + 8), W2(g, 2 * tq + 9), f[1], f[3]);
  fq[32 * 4] = make_uint4(f[0], f[1], f[2], f[3]);
  fq[32 * 5] = make_uint4(w2b[0], w2b[1], w2b[2], w2b[3]);
  F.b2[0] = ws[L::B2S + 2 * tq];  // zero beyond the 3 outputs
  F.b2[1] = ws[L::B2S + 2 * tq + 1];
}

// A fragment (hi, lo) of a 16 x 16 activation tile held as two n-tile accumulators
__device__ __forceinline__ void frag_a(const float (&v)[2][4], uint32_t (&hi)[4], uint32_t (&lo)[4]) {
  pack_act<true>(v[0][0], v[0][1], hi[0], lo[0]);
  pack_act<true>(v[0][2], v[0][3], hi[1], lo[1]);
  pack_act<true>(v[1][0], v[1][1], hi[2], lo[2]);
  pack_act<true>(v[1][2], v[1][3], hi[3], lo[3]);
}

// c += A * B in three bf16 passes (B given as {b0 hi, b1 hi, b0 lo, b1 lo})
__device__ __forceinline__ void mma3(float (&c)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4], uint4 b) {
  mma16816(c, ah, b.x, b.y);
  mma16816(c, al, b.x, b.y);
  mma16816(c, ah, b.z, b.w);
}

// Transpose of an 8 x 8 bf16 block held one row per 4 lanes (C / A fragment
// quarter) into the B-fragment orientation: lane (g, tq) receives rows
// 2tq, 2tq+1 of column g.
__device__ __forceinline__ uint32_t movt(uint32_t x) {
  uint32_t y;
  asm("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// Per-warp gradient sums of one step, as MMA accumulators (K = pixels):
//   w1[j]: gW1 | gb1 = d1^T [a0 | 1]  rows o = g + 8(e>>1), cols k = 8j + 2tq + (e&1)
//   w2t:   (gW2 | gb2)^T = [a1 | 1]^T d2  rows k, cols output j
//   w0:    gW0 | gb0 = d0^T [x y 1]   rows o, cols (x, y, 1)
struct FitGrads {
  float w1[2][4], w2t[4], w0[4];
};

// {A^T} of a 16 x 16 tile given as A-fragment words (rows = pixels): the
// A fragment of its transpose (rows = units, K = pixels)
__device__ __forceinline__ void frag_at(const uint32_t (&p)[4], uint32_t (&t)[4]) {
  t[0] = movt(p[0]);
  t[1] = movt(p[2]);
  t[2] = movt(p[1]);
  t[3] = movt(p[3]);
}

// MT m-tiles (16 MT pixels from px0) of one step: the loss into lp and, when
// bwd, this tile's outer products into G.  xyt / tgt: per-pixel coordinate
// and target tables (images up to kPixTable pixels), else colx / rowy.
template <int H, int MT>
__device__ __forceinline__ void mma_pass(const FitFrags& F, const uint4* fq, const FitArgs& A, const float* __restrict__ img,
                                         const float2* xyt, const float4* tgt, const float* colx,
                                         const float* rowy, float inv_wd, int px0, float om,
                                         float s2, bool bwd, int lane, double& lp, FitGrads& G) {
  const int g = lane >> 2, tq = lane & 3;
  float x[MT][2], y[MT][2], tg[MT][2][2];
  bool ok[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int px = px0 + 16 * mt + g + 8 * h;
      ok[mt][h] = px < A.hw;
      if (xyt) {
        const float2 c = ok[mt][h] ? xyt[px] : make_float2(0.0f, 0.0f);
        const float2 t = ok[mt][h] && tq < 2 ? reinterpret_cast<const float2*>(tgt + px)[tq] : make_float2(0.0f, 0.0f);
        x[mt][h] = c.x;
        y[mt][h] = c.y;
        tg[mt][h][0] = t.x;
        tg[mt][h][1] = t.y;
        continue;
      }
      int pr = int(float(px) * inv_wd), pc = px - pr * A.wd;  // exact after one correction
      if (pc < 0) {
        --pr;
        pc += A.wd;
      } else if (pc >= A.wd) {
        ++pr;
        pc -= A.wd;
      }
      if (!ok[mt][h]) pr = pc = 0;
      x[mt][h] = colx[pc];
      y[mt][h] = rowy[pr];
#pragma unroll
      for (int e = 0; e < 2; ++e)
        tg[mt][h][e] = ok[mt][h] && 2 * tq + e < 3 ? img[3 * px + 2 * tq + e] : 0.0f;
    }
  float lpf = 0.0f;  // this pass's squared residuals (f32 partial, added to the f64 total below)
  // per-lane unit masks: keep = 1 for real units, one = 1 at the ones column
  // (unit H).  Pad units need no mask in the backward: their B columns are 0.
  float keep[2][2], one[2][2];
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int u = 8 * j + 2 * tq + e;
      keep[j][e] = u < H ? 1.0f : 0.0f;
      one[j][e] = u == H ? 1.0f : 0.0f;
    }
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    // layer 0 (FFMA, fragment layout)
    float v[2][4], c0[2][4];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = e >> 1;
        const float z = fmaf(x[mt][h], F.w0x[j][e & 1], fmaf(y[mt][h], F.w0y[j][e & 1], F.b0[j][e & 1]));
        float sn;
        __sincosf(z, &sn, &c0[j][e]);  // z already carries omega
        v[j][e] = fmaf(sn, keep[j][e & 1], one[j][e & 1]);
      }
    uint32_t a0h[4], a0l[4];
    frag_a(v, a0h, a0l);
    // layer 1
    float c1[2][4];
    {
      float z[2][4];  // accumulators start at the bias
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) z[j][e] = F.b1[j][e & 1];
#pragma unroll
      for (int j = 0; j < 2; ++j) mma3(z[j], a0h, a0l, frag_ld(fq + 32 * j));
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float sn;
          __sincosf(z[j][e], &sn, &c1[j][e]);
          v[j][e] = fmaf(sn, keep[j][e & 1], one[j][e & 1]);
        }
    }
    uint32_t a1h[4], a1l[4];
    frag_a(v, a1h, a1l);
    // layer 2, residual, loss, d2 = (2 / size) * resid
    float d2[4];
    {
      float o[4] = {F.b2[0], F.b2[1], F.b2[0], F.b2[1]};
      mma3(o, a1h, a1l, frag_ld(fq + 32 * 4));
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = e >> 1;
        const bool val = ok[mt][h] && 2 * tq + (e & 1) < 3;
        const float r = __fsub_rn(o[e], tg[mt][h][e & 1]);
        if (val) lpf = fmaf(r, r, lpf);
        d2[e] = val ? __fmul_rn(s2, r) : 0.0f;
      }
    }
    if (!bwd) continue;
    // d1 = (d2 W2) * c1: A = d2 (K = output j; columns >= 8 zero)
    uint32_t d2h[4] = {0u, 0u, 0u, 0u}, d2l[4] = {0u, 0u, 0u, 0u};
    pack_act<true>(d2[0], d2[1], d2h[0], d2l[0]);
    pack_act<true>(d2[2], d2[3], d2h[1], d2l[1]);
    {
      float q[2][4] = {};
      const uint4 w = frag_ld(fq + 32 * 5);
      mma16816(q[0], d2h, w.x, 0u);
      mma16816(q[1], d2h, w.z, 0u);
      mma16816(q[0], d2l, w.x, 0u);
      mma16816(q[1], d2l, w.z, 0u);
      mma16816(q[0], d2h, w.y, 0u);
      mma16816(q[1], d2h, w.w, 0u);
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) c1[j][e] = __fmul_rn(q[j][e], c1[j][e]);  // c1 := d1
    }
    uint32_t d1h[4], d1l[4];
    frag_a(c1, d1h, d1l);
    // d0 = (d1 W1) * c0
    {
      float r[2][4] = {};
#pragma unroll
      for (int j = 0; j < 2; ++j) mma3(r[j], d1h, d1l, frag_ld(fq + 32 * (2 + j)));
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) c0[j][e] = __fmul_rn(r[j][e], c0[j][e]);  // c0 := d0
    }
    // gradient sums over this tile's 16 pixels (bf16 3-pass, K = pixels)
    {
      uint32_t th[4], tl[4], bh[4], bl[4];
      frag_at(d1h, th);  // A = d1^T
      frag_at(d1l, tl);
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // B = [a0 | 1]: n-tile j = words 2j, 2j+1
        bh[i] = movt(a0h[i]);
        bl[i] = movt(a0l[i]);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        mma16816(G.w1[j], th, bh[2 * j], bh[2 * j + 1]);
        mma16816(G.w1[j], tl, bh[2 * j], bh[2 * j + 1]);
        mma16816(G.w1[j], th, bl[2 * j], bl[2 * j + 1]);
      }
      frag_at(a1h, th);  // A = [a1 | 1]^T, B = d2
      frag_at(a1l, tl);
      const uint32_t e0h = movt(d2h[0]), e1h = movt(d2h[1]), e0l = movt(d2l[0]), e1l = movt(d2l[1]);
      mma16816(G.w2t, th, e0h, e1h);
      mma16816(G.w2t, tl, e0h, e1h);
      mma16816(G.w2t, th, e0l, e1l);
      uint32_t d0h[4], d0l[4];
      frag_a(c0, d0h, d0l);
      frag_at(d0h, th);  // A = d0^T, B = [x y 1] of pixels 2tq, 2tq+1 (+8)
      frag_at(d0l, tl);
      float xb[4], yb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int src = 4 * (2 * tq + (i & 1));  // lane holding pixel row 2tq + (i&1) (+8 for i >= 2)
        xb[i] = __shfl_sync(0xffffffffu, x[mt][i >> 1], src);
        yb[i] = __shfl_sync(0xffffffffu, y[mt][i >> 1], src);
      }
      auto col = [&](int i) { return g == 0 ? xb[i] : (g == 1 ? yb[i] : (g == 2 ? 1.0f : 0.0f)); };
      uint32_t b0h, b0l, b1h, b1l;
      pack_act<true>(col(0), col(1), b0h, b0l);
      pack_act<true>(col(2), col(3), b1h, b1l);
      mma16816(G.w0, th, b0h, b1h);
      mma16816(G.w0, tl, b0h, b1h);
      mma16816(G.w0, th, b0l, b1l);
    }
  }
  lp += double(lpf);
}

// Write a warp's step sums into its partial row (canonical order).  Every
// entry of the row has exactly one owner lane, so plain stores suffice (no
// zeroing, no read-modify-write).
template <int H>
__device__ __forceinline__ void fold_grads(const FitGrads& G, float* pw, int lane) {
  using L = FitLayout<H>;
  const int g = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = g + 8 * (e >> 1), cb = 2 * tq + (e & 1);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = 8 * j + cb;
      if (r < H) {
        if (k < H) pw[2 * H + r * H + k] = G.w1[j][e];
        else if (k == H) pw[L::P + H + r] = G.w1[j][e];
      }
    }
    if (cb < 3) {
      if (r < H) pw[2 * H + H * H + cb * H + r] = G.w2t[e];
      else if (r == H) pw[L::P + 2 * H + cb] = G.w2t[e];
    }
    if (r < H) {
      if (cb < 2) pw[2 * r + cb] = G.w0[e];
      else if (cb == 2) pw[L::P + r] = G.w0[e];
    }
  }
}

#ifndef RINR_FIT_MINB
#define RINR_FIT_MINB 2  // CTAs per SM the MMA pass is compiled for (128 registers)
#endif
#ifndef RINR_FIT_MT
#define RINR_FIT_MT 2  // m-tiles per MMA pass
#endif
template <int H, bool ACC, int NPX, bool MMA>
__global__ void __launch_bounds__(kFitThreads / NPX, MMA ? RINR_FIT_MINB : 1) fit_kernel(FitArgs A) {
  static_assert(!MMA || (!ACC && H < 16), "tensor-core pixel pass: MUFU sine, H < 16");
  using L = FitLayout<H>;
  constexpr int NWP = kFitWarps / NPX;         // warps per CTA
  constexpr int NTH = NWP * 32;                // threads per CTA
  constexpr int CPX = 32 * NPX;                // pixels per warp chunk
  extern __shared__ __align__(16) float sm[];
  float* ws = sm;
  float* mo = ws + L::WS;
  float* ve = mo + L::NPAR_PAD;
  float* mk = ve + L::NPAR_PAD;
  float* part = mk + ((L::P + 3) & ~3);
  float* stage = part + NWP * L::NPAR_PAD;
  double* lossw = reinterpret_cast<double*>(stage + (MMA ? 0 : NWP * CPX * kStage));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint4* frg = reinterpret_cast<uint4*>(lossw + kFitWarps) + warp * kFragGroups * 32 + lane;  // MMA pass
  // MMA pass tables: per-pixel (x, y) and (r, g, b, 0) when hw <= kPixTable, else per-axis coordinates
  char* tab = reinterpret_cast<char*>(reinterpret_cast<uint4*>(lossw + kFitWarps) + NWP * kFragGroups * 32);
  const bool pixtab = A.hw <= kPixTable;
  float2* xyt = pixtab ? reinterpret_cast<float2*>(tab) : nullptr;
  float4* tgt = pixtab ? reinterpret_cast<float4*>(tab + ((size_t(A.hw) * 8 + 15) & ~size_t(15))) : nullptr;
  float* colx = reinterpret_cast<float*>(tab);
  float* rowy = colx + A.wd;
  const int64_t m = blockIdx.x;
  float* gw = A.w + m * L::P;
  float* gb = A.b + m * L::PB;

  for (int i = tid; i < L::WS; i += NTH) ws[i] = 0.0f;
  __syncthreads();
  for (int p = tid; p < L::NPAR; p += NTH) {
    L::put(ws, p, p < L::P ? gw[p] : gb[p - L::P]);
    mo[p] = 0.0f;
    ve[p] = 0.0f;
    if (p < L::P) mk[p] = A.mask[m * L::P + p] ? 1.0f : 0.0f;
  }
  if constexpr (MMA) {
    if (pixtab) {
      const float* im = A.images + m * int64_t(A.hw) * 3;
      for (int i = tid; i < A.hw; i += NTH) {
        const int r = i / A.wd, c = i - r * A.wd;
        xyt[i] = make_float2(grid_coord(c, A.wd, A.inv_wm1), grid_coord(r, A.h, A.inv_hm1));
        tgt[i] = make_float4(im[3 * i], im[3 * i + 1], im[3 * i + 2], 0.0f);
      }
    } else {
      for (int i = tid; i < A.wd; i += NTH) colx[i] = grid_coord(i, A.wd, A.inv_wm1);
      for (int i = tid; i < A.h; i += NTH) rowy[i] = grid_coord(i, A.h, A.inv_hm1);
    }
  }
  __syncthreads();
  const float inv_wd = 1.0f / float(A.wd);

  const int HW = A.hw, nchunks = (HW + CPX - 1) / CPX;
  const double scale = 1.0 / (3.0 * double(HW));  // 1.0 / resid.size
  const float s2 = float(2.0 * scale);
  const float om = float(A.omega);
  const int stride = A.steps / 64 > 1 ? A.steps / 64 : 1;
  const float* img = A.images + m * int64_t(HW) * 3;
  float* st = stage + warp * CPX * kStage;
  const int o16 = lane & 15;
  const bool hi_half = lane >= 16;
  int slot_c = 0;
  int32_t status = 0;

  for (int t = 0; t <= A.steps; ++t) {
    // t == steps: the final forward-only loss (encoder.py:84), except for the
    // loss_and_grad hook (steps == 0 with gradient outputs)
    const bool last = t == A.steps && !(A.grad_w && A.steps == 0);
    FitFrags F;
    FitGrads G = {};
    if constexpr (MMA) {
      load_frags<H>(ws, lane, om, F, frg);  // this step's weights as MMA B fragments
      __syncwarp();
    }
    // this warp's partial gradient row (canonical order), summed over its chunks
    float* pw = part + warp * L::NPAR_PAD;
    if (!last && !MMA)
      for (int i = lane; i < L::NPAR_PAD; i += 32) pw[i] = 0.0f;
    __syncwarp();
    double lp = 0.0;
    for (int ch = warp; ch < nchunks; ch += NWP) {
      if constexpr (MMA) {
        constexpr int MT = RINR_FIT_MT;
#pragma unroll 1
        for (int q = 0; q < CPX; q += 16 * MT)
          mma_pass<H, MT>(F, frg, A, img, xyt, tgt, colx, rowy, inv_wd, ch * CPX + q, om, s2, !last, lane, lp, G);
        continue;  // the gradient sums stay in G until the end of the step
      } else {
      float x[NPX], y[NPX], tg[NPX][3];
      bool valid[NPX];
#pragma unroll
      for (int p = 0; p < NPX; ++p) {
        const int px = ch * CPX + p * 32 + lane;
        valid[p] = px < HW;
        const int pr = valid[p] ? px / A.wd : 0, pc = valid[p] ? px - pr * A.wd : 0;
        x[p] = grid_coord(pc, A.wd, A.inv_wm1);
        y[p] = grid_coord(pr, A.h, A.inv_hm1);
        tg[p][0] = tg[p][1] = tg[p][2] = 0.0f;
        if (valid[p]) {
          tg[p][0] = img[3 * px];
          tg[p][1] = img[3 * px + 1];
          tg[p][2] = img[3 * px + 2];
        }
      }
      float a0[NPX][16], c0[NPX][16], a1[NPX][16], c1[NPX][16], d2[NPX][3], out[NPX][3];
      double lpx[NPX];
#pragma unroll
      for (int p = 0; p < NPX; ++p) lpx[p] = 0.0;
      pixel_pass<H, ACC, true, NPX>(ws, x, y, tg, om, s2, a0, c0, a1, c1, d2, out, lpx);
#pragma unroll
      for (int p = 0; p < NPX; ++p)
        if (valid[p]) lp += lpx[p];
      if (last) continue;
#pragma unroll
      for (int p = 0; p < NPX; ++p) {
        if (!valid[p]) {
#pragma unroll
          for (int k = 0; k < 16; ++k) c0[p][k] = c1[p][k] = 0.0f;
          d2[p][0] = d2[p][1] = d2[p][2] = 0.0f;
        }
        float* row = st + (p * 32 + lane) * kStage;
#pragma unroll
        for (int k = 0; k < 16; k += 4) {
          *reinterpret_cast<float4*>(row + SA0 + k) = make_float4(a0[p][k], a0[p][k + 1], a0[p][k + 2], a0[p][k + 3]);
          *reinterpret_cast<float4*>(row + SA1 + k) = make_float4(a1[p][k], a1[p][k + 1], a1[p][k + 2], a1[p][k + 3]);
          *reinterpret_cast<float4*>(row + SD1 + k) = make_float4(c1[p][k], c1[p][k + 1], c1[p][k + 2], c1[p][k + 3]);
          *reinterpret_cast<float4*>(row + SD0 + k) = make_float4(c0[p][k], c0[p][k + 1], c0[p][k + 2], c0[p][k + 3]);
        }
        *reinterpret_cast<float4*>(row + SD2) = make_float4(d2[p][0], d2[p][1], d2[p][2], 0.0f);
        *reinterpret_cast<float4*>(row + SXY) = make_float4(x[p], y[p], 1.0f, 0.0f);
        if constexpr (H < 16) {  // ones column: the tensor-core reduction also yields the bias gradients
          row[SA0 + H] = 1.0f;
          row[SA1 + H] = 1.0f;
        }
      }
      }
      __syncwarp();
      const int nq = HW - ch * CPX < CPX ? HW - ch * CPX : CPX;
      if constexpr (H < 16) {
        tc_reduce<H>(st, CPX, pw, lane);
      } else {
      // per-lane accumulators live only for this chunk (uniform stream, see header)
        float g8[8], g3[3], gq[3], gp = 0.0f, gu = 0.0f;
  #pragma unroll
        for (int k = 0; k < 8; ++k) g8[k] = 0.0f;
  #pragma unroll
        for (int j = 0; j < 3; ++j) g3[j] = gq[j] = 0.0f;
        // lanes < 16: u = d1[o], vec = a0[0..7], p = d0[o], q = (x, y, 0)
        // lanes >= 16: u = d1[o], vec = a0[8..15], p = a1[o], q = d2[0..2]
        const int vo = hi_half ? SA0 + 8 : SA0;
        const int po = hi_half ? SA1 + o16 : SD0 + o16;
        const int qo = hi_half ? SD2 : SXY;
        for (int q = 0; q < nq; ++q) {
          const float* r = st + q * kStage;
          const float u = r[SD1 + o16];
          const float4 v0 = *reinterpret_cast<const float4*>(r + vo);
          const float4 v1 = *reinterpret_cast<const float4*>(r + vo + 4);
          const float p = r[po];
          const float4 qq = *reinterpret_cast<const float4*>(r + qo);
          g8[0] = fmaf(u, v0.x, g8[0]);
          g8[1] = fmaf(u, v0.y, g8[1]);
          g8[2] = fmaf(u, v0.z, g8[2]);
          g8[3] = fmaf(u, v0.w, g8[3]);
          g8[4] = fmaf(u, v1.x, g8[4]);
          g8[5] = fmaf(u, v1.y, g8[5]);
          g8[6] = fmaf(u, v1.z, g8[6]);
          g8[7] = fmaf(u, v1.w, g8[7]);
          g3[0] = fmaf(p, qq.x, g3[0]);
          g3[1] = fmaf(p, qq.y, g3[1]);
          g3[2] = fmaf(p, qq.z, g3[2]);
          gp += p;
          gu += u;
          gq[0] += qq.x;
          gq[1] += qq.y;
          gq[2] += qq.z;
        }
        // fold into the warp's partial row; every canonical entry has one owner lane
        {
          const int o = o16;
          if (o < H) {
            if (!hi_half) {
  #pragma unroll
              for (int k = 0; k < 8; ++k)
                if (k < H) pw[2 * H + o * H + k] += g8[k];
              pw[2 * o] += g3[0];
              pw[2 * o + 1] += g3[1];
              pw[L::P + o] += gp;      // b0
              pw[L::P + H + o] += gu;  // b1
            } else {
  #pragma unroll
              for (int k = 0; k < 8; ++k)
                if (8 + k < H) pw[2 * H + o * H + 8 + k] += g8[k];
  #pragma unroll
              for (int j = 0; j < 3; ++j) pw[2 * H + H * H + j * H + o] += g3[j];
              if (o == 0)
  #pragma unroll
                for (int j = 0; j < 3; ++j) pw[L::P + 2 * H + j] += gq[j];
            }
          }
        }
  
      }
      __syncwarp();
    }
    if constexpr (MMA)
      if (!last) fold_grads<H>(G, pw, lane);
    // loss of this step (weights before the update)
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, d);
    if (lane == 0) lossw[warp] = lp;
    __syncthreads();
    double loss = 0.0;
    for (int i = 0; i < NWP; ++i) loss += lossw[i];
    loss *= scale;
    if (!isfinite(loss)) {
      status = t + 1;
      break;
    }
    if (tid == 0 && (t % stride == 0 || t == A.steps) && slot_c < A.cap) A.curve[m * A.cap + slot_c++] = loss;
    if (t == 0 && A.grad_w && !last) {
      for (int p = tid; p < L::NPAR; p += NTH) {
        float g = 0.0f;
        for (int i = 0; i < NWP; ++i) g += part[i * L::NPAR_PAD + p];
        if (p < L::P) A.grad_w[m * L::P + p] = __fmul_rn(g, mk[p]);
        else A.grad_b[m * L::PB + p - L::P] = g;
      }
      if (tid == 0) A.loss0[m] = loss;
      if (A.steps == 0) break;
    }
    if (t == A.steps) break;
    // Adam step (net.py:282-296), numpy's f32 operation order
    float lr, c1, c2;
    if (A.sched) {
      lr = A.sched[3 * t];
      c1 = A.sched[3 * t + 1];
      c2 = A.sched[3 * t + 2];
    } else {
      c1 = float(1.0 - pow(0.9, double(t + 1)));
      c2 = float(1.0 - pow(0.999, double(t + 1)));
      lr = float(0.5 * A.lr0 * (1.0 + cos(3.141592653589793 * double(t) / double(A.steps))));
    }
    for (int p = tid; p < L::NPAR; p += NTH) {
      float g = 0.0f;
      for (int i = 0; i < NWP; ++i) g += part[i * L::NPAR_PAD + p];
      if (p < L::P) g = __fmul_rn(g, mk[p]);  // gw * mask
      float mp = __fadd_rn(__fmul_rn(mo[p], 0.9f), __fmul_rn(float(1.0 - 0.9), g));
      float vp = __fadd_rn(__fmul_rn(ve[p], 0.999f), __fmul_rn(__fmul_rn(float(1.0 - 0.999), g), g));
      mo[p] = mp;
      ve[p] = vp;
      const int s = L::slot(p);
      const float upd = __fdiv_rn(__fmul_rn(lr, __fdiv_rn(mp, c1)), __fadd_rn(__fsqrt_rn(__fdiv_rn(vp, c2)), 1e-8f));
      float w = __fsub_rn(ws[s], upd);
      if (p < L::P) w = __fmul_rn(w, mk[p]);  // np.multiply(layer.w, mask)
      L::put(ws, p, w);
    }
    __syncthreads();
  }
  __syncthreads();
  for (int p = tid; p < L::NPAR; p += NTH) {
    const float v = ws[L::slot(p)];
    if (p < L::P) gw[p] = v;
    else gb[p - L::P] = v;
  }
  if (tid == 0) {
    A.status[m] = status;
    for (int s = slot_c; s < A.cap; ++s) A.curve[m * A.cap + s] = NAN;
  }
}

template <int H, bool ACC>
__global__ void __launch_bounds__(256) render_kernel(int64_t n, const float* __restrict__ w,
                                                     const float* __restrict__ b, int h, int wd, double inv_wm1,
                                                     double inv_hm1, float om, float* __restrict__ out) {
  using L = FitLayout<H>;
  __shared__ __align__(16) float ws[L::WS];
  const int64_t m = blockIdx.y;
  for (int i = threadIdx.x; i < L::WS; i += 256) ws[i] = 0.0f;
  __syncthreads();
  for (int p = threadIdx.x; p < L::NPAR; p += 256) L::put(ws, p, p < L::P ? w[m * L::P + p] : b[m * L::PB + p - L::P]);
  __syncthreads();
  const int HW = h * wd;
  const int px = blockIdx.x * 256 + threadIdx.x;
  if (px >= HW) return;
  const int pr = px / wd, pc = px - pr * wd;
  const float x = grid_coord(pc, wd, inv_wm1), y = grid_coord(pr, h, inv_hm1);
  float a0[1][16], c0[1][16], a1[1][16], c1[1][16], d2[1][3], o[1][3], tg[1][3] = {{0.f, 0.f, 0.f}};
  double lp[1] = {0.0};
  const float xs[1] = {x}, ys[1] = {y};
  pixel_pass<H, ACC, false, 1>(ws, xs, ys, tg, om, 0.0f, a0, c0, a1, c1, d2, o, lp);
  float* dst = out + (m * HW + px) * 3;
#pragma unroll
  for (int j = 0; j < 3; ++j) dst[j] = fminf(fmaxf(o[0][j], 0.0f), 1.0f);  // np.clip(rgb, 0, 1)
}

int fit_arch(const int32_t* dims, int nl, int& H) {
  if (!dims || nl != 3 || dims[0] != 2 || dims[3] != 3 || dims[1] != dims[2] || dims[1] < 8 || dims[1] > 16)
    return set_error(RINR_ERR_UNSUPPORTED, "the GPU encoder supports architectures (2, H, H, 3) with 8 <= H <= 16");
  H = dims[1];
  return RINR_OK;
}

template <int H, bool ACC, int NPX, bool MMA>
int launch_fit(const FitArgs& a, cudaStream_t st) {
  constexpr size_t smem0 = FitLayout<H>::smem_bytes(NPX, !MMA);
  static_assert(smem0 <= 227 * 1024, "fit kernel shared memory");
  const size_t tabs = a.hw <= kPixTable ? ((size_t(a.hw) * 8 + 15) & ~size_t(15)) + size_t(a.hw) * 16
                                        : sizeof(float) * size_t(a.h + a.wd);
  const size_t smem = smem0 + (MMA ? tabs : 0);
  if (smem > 227 * 1024) return set_error(RINR_ERR_UNSUPPORTED, "fit: image too large for the coordinate tables");
  // the shared-memory limit is a per-device attribute: raise it once per device
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(RINR_ERR_CUDA, "fit: no current device");
  const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
  if (!(attr_done.load() & bit)) {
    if (cudaFuncSetAttribute(fit_kernel<H, ACC, NPX, MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
        cudaSuccess)
      return set_error(RINR_ERR_CUDA, "fit smem attribute");
    attr_done.fetch_or(bit);
  }
  fit_kernel<H, ACC, NPX, MMA><<<unsigned(a.n), kFitThreads / NPX, smem, st>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(RINR_ERR_CUDA, std::string("fit launch: ") + cudaGetErrorString(e));
  return RINR_OK;
}

// two pixels per thread (8 warps): each weight row from shared memory
// serves two pixels (one pixel per thread with 16 warps measured 6% slower)
template <int H>
int dispatch_fit(const FitArgs& a, bool acc, cudaStream_t st) {
  if (acc) return launch_fit<H, true, RINR_FIT_NPX, false>(a, st);
  // MUFU mode: tensor-core pixel pass (H < 16; RINR_FIT_FFMA builds the fp32 FFMA pass instead)
#ifndef RINR_FIT_FFMA
  if constexpr (H < 16) return launch_fit<H, false, RINR_FIT_NPX, true>(a, st);
#endif
  return launch_fit<H, false, RINR_FIT_NPX, false>(a, st);
}

template <int H, bool ACC>
int launch_render(int64_t n, const float* w, const float* b, int h, int wd, double om, float* out, cudaStream_t st) {
  const dim3 grid(unsigned((h * wd + 255) / 256), unsigned(n));
  render_kernel<H, ACC><<<grid, 256, 0, st>>>(n, w, b, h, wd, wd > 1 ? 1.0 / double(wd - 1) : 0.0,
                                              h > 1 ? 1.0 / double(h - 1) : 0.0, float(om), out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(RINR_ERR_CUDA, std::string("render launch: ") + cudaGetErrorString(e));
  return RINR_OK;
}

}  // namespace
}  // namespace rinr

using namespace rinr;

// General architectures (fit_general.cu)
int rinr_fit_general(const int32_t* dims, int nl, int64_t n, float* d_w, float* d_b, const uint8_t* d_mask,
                     const float* d_images, const rinr_fit_params_t* p, double* d_curve, int32_t* d_status,
                     float* d_grad_w, float* d_grad_b, double* d_loss0, void* stream);
int rinr_fit_render_general(const int32_t* dims, int nl, int64_t n, const float* d_w, const float* d_b, int32_t h,
                            int32_t w, double omega, int32_t sin_mode, float* d_out, void* stream);

static bool narrow_arch(const int32_t* dims, int nl) {
  return dims && nl == 3 && dims[0] == 2 && dims[3] == 3 && dims[1] == dims[2] && dims[1] >= 8 && dims[1] <= 16;
}

extern "C" int rinr_fit(const int32_t* dims, int nl, int64_t n, float* d_w, float* d_b, const uint8_t* d_mask,
                        const float* d_images, const rinr_fit_params_t* p, double* d_curve, int32_t* d_status,
                        float* d_grad_w, float* d_grad_b, double* d_loss0, void* stream) {
  clear_error();
  if (!p || n < 0) return set_error(RINR_ERR_INVALID_INPUT, "null params or negative n");
  if (p->h < 1 || p->w < 1 || p->steps < 0 || p->curve_cap < 1) return set_error(RINR_ERR_INVALID_INPUT, "bad fit params");
  if (n == 0) return RINR_OK;
  if (!d_w || !d_b || !d_mask || !d_images || !d_curve || !d_status)
    return set_error(RINR_ERR_INVALID_INPUT, "null buffer");
  if ((d_grad_w == nullptr) != (d_grad_b == nullptr) || (d_grad_w && !d_loss0))
    return set_error(RINR_ERR_INVALID_INPUT, "grad outputs need d_grad_w, d_grad_b and d_loss0");
  if (!narrow_arch(dims, nl))  // deep / wide nets: the general per-step kernels
    return rinr_fit_general(dims, nl, n, d_w, d_b, d_mask, d_images, p, d_curve, d_status, d_grad_w, d_grad_b,
                            d_loss0, stream);
  int H = 0;
  if (int e = fit_arch(dims, nl, H)) return e;
  FitArgs a{};
  a.n = n;
  a.w = d_w;
  a.b = d_b;
  a.mask = d_mask;
  a.images = d_images;
  a.h = p->h;
  a.wd = p->w;
  a.hw = p->h * p->w;
  a.steps = p->steps;
  a.cap = p->curve_cap;
  a.inv_wm1 = p->w > 1 ? 1.0 / double(p->w - 1) : 0.0;
  a.inv_hm1 = p->h > 1 ? 1.0 / double(p->h - 1) : 0.0;
  a.lr0 = p->lr0;
  a.omega = p->omega;
  a.curve = d_curve;
  a.status = d_status;
  a.grad_w = d_grad_w;
  a.grad_b = d_grad_b;
  a.loss0 = d_loss0;
  a.sched = p->sched;
  const bool acc = p->sin_mode == RINR_SIN_ACCURATE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (H) {
#define RINR_FIT_CASE(HH) \
  case HH:                \
    return dispatch_fit<HH>(a, acc, st);
    RINR_FIT_CASE(8) RINR_FIT_CASE(9) RINR_FIT_CASE(10) RINR_FIT_CASE(11) RINR_FIT_CASE(12)
    RINR_FIT_CASE(13) RINR_FIT_CASE(14) RINR_FIT_CASE(15) RINR_FIT_CASE(16)
#undef RINR_FIT_CASE
    default: return set_error(RINR_ERR_UNSUPPORTED, "GPU encoder: hidden width must be 8..16");
  }
}

extern "C" int rinr_fit_render(const int32_t* dims, int nl, int64_t n, const float* d_w, const float* d_b, int32_t h,
                               int32_t w, double omega, int32_t sin_mode, float* d_out, void* stream) {
  clear_error();
  if (n < 0 || h < 1 || w < 1) return set_error(RINR_ERR_INVALID_INPUT, "bad render size");
  if (n == 0) return RINR_OK;
  if (!d_w || !d_b || !d_out) return set_error(RINR_ERR_INVALID_INPUT, "null buffer");
  if (!narrow_arch(dims, nl)) return rinr_fit_render_general(dims, nl, n, d_w, d_b, h, w, omega, sin_mode, d_out, stream);
  int H = 0;
  if (int e = fit_arch(dims, nl, H)) return e;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool acc = sin_mode == RINR_SIN_ACCURATE;
  switch (H) {
#define RINR_RENDER_CASE(HH)                                                   \
  case HH:                                                                     \
    return acc ? launch_render<HH, true>(n, d_w, d_b, h, w, omega, d_out, st)  \
               : launch_render<HH, false>(n, d_w, d_b, h, w, omega, d_out, st);
    RINR_RENDER_CASE(8) RINR_RENDER_CASE(9) RINR_RENDER_CASE(10) RINR_RENDER_CASE(11) RINR_RENDER_CASE(12)
    RINR_RENDER_CASE(13) RINR_RENDER_CASE(14) RINR_RENDER_CASE(15) RINR_RENDER_CASE(16)
#undef RINR_RENDER_CASE
    default: return set_error(RINR_ERR_UNSUPPORTED, "GPU encoder: hidden width must be 8..16");
  }
}
