// Uniform-width SIREN decode on mma.sync.m16n8k16 (bf16 operands, f32
// accumulate), register-resident layer chain.
//
// Work unit: one warp evaluates NB blocks of 16 consecutive pixels of one
// image.  Per block and hidden layer the warp holds the activation tile as
// bf16 A fragments; the f32 accumulator fragments of n-tiles 2t and 2t+1 are
// exactly the A fragment of k-tile t of the next layer, so
// MMA -> scale/bias FFMA -> sine -> bf16 pack -> next MMA stays in registers.
//
// Numerics (reference net.py:190-201 is z = a @ w.T + b; a = sin(omega z)):
//   * omega is folded into weights/biases/scales in the prologue.
//   * Hidden layers stored as affine8 codes (archive.py:294-301) use the
//     integer (code - zero_point) as the B operand — exact in bf16 — and apply
//     f32(omega * scale) after the MMA, so the weights need no hi/lo split.
//     Other layers use B = omega * w split into bf16 hi + lo.
//   * X3 (precision FP32): A split into bf16 hi + lo (both round-to-nearest), products
//     Ah*Bh + Al*Bh (+ Ah*Bl for float B); max-abs vs the CPU oracle ~1e-5.
//   * BF16: one pass.
//   * Output layer: bias add + clamp in one saturating FADD (decoder.py:35).
//     Crop padding enters as NaN coordinates; saturate maps NaN to 0, the
//     zero fill the epilogue specification asks for.
#pragma once

#include "device_common.cuh"

namespace rinr {

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// d = A * B (zero accumulator: the C operand is RZ, no register moves)
__device__ __forceinline__ void mma16816_z(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%10,%10,%10};\n"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(0.0f));
}

__device__ __forceinline__ uint32_t bf2_bits(__nv_bfloat162 v) { return *reinterpret_cast<uint32_t*>(&v); }

// Blackwell packed fp32 (FFMA2 / FADD2): two IEEE fp32 ops, each rounded as
// the scalar op would be, in one issue slot.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\tmov.b64 rc, {%6,%7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2_(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2,%3};\n\tmov.b64 rb, {%4,%5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// (x0, x1) -> packed bf16x2 hi = RN(x) and, for the split, lo = RN(x - hi):
// |x - hi - lo| <= 2^-18 |x|.  Four instructions per pair: F2FP packs hi,
// two FHFMA.BF16 form x - hi exactly in f32 straight from the packed bf16
// halves (the sm_100 mixed-precision fma.rn.f32.bf16, hi * -1 + x), F2FP packs lo.
template <bool X3>
__device__ __forceinline__ void pack_act(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(x1), "f"(x0));
  if constexpr (X3) {
    float l0, l1;
    const unsigned short neg_one = 0xBF80;  // bf16 -1.0, a loop-invariant register
    asm("{.reg .b16 h0, h1;\n\tmov.b32 {h0, h1}, %2;\n\t"
        "fma.rn.f32.bf16 %0, h0, %5, %3;\n\tfma.rn.f32.bf16 %1, h1, %5, %4;}"
        : "=f"(l0), "=f"(l1)
        : "r"(hi), "f"(x0), "f"(x1), "h"(neg_one));
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(l1), "f"(l0));
  }
}

template <bool ACCURATE>
__device__ __forceinline__ float sine(float x) {
  if constexpr (ACCURATE) return sinf(x);
  return __sinf(x);
}

// Shared-memory image of one record's network, zero padded to the MMA tiles.
//   fragH[h][t][j][lane] uint4 {b0 hi, b1 hi, b0 lo, b1 lo} of hidden layer h+1
//   fragO[t][lane]       uint4, last layer (n-tile 0; output c in column 2c, persist.cuh)
//   l0[c]                float4 {omega w[c][0], omega w[c][1], omega b[c], 0}
//   biasH[h][c]          omega * b;   scaleH[h]: f32(omega*scale) or 1
//   modeH[h]             1 = integer-code B (affine8), 0 = float B split
//   biasO[8]
template <int HID, int NL>
struct MmaCfg {
  static constexpr int KP = (HID + 15) / 16 * 16;
  static constexpr int KT = KP / 16;
  static constexpr int NT = (HID + 7) / 8;
  static constexpr int NH = NL - 2;
  static constexpr int FRAG_H = NH * KT * NT * 32 * 4;  // u32 words
  static constexpr int FRAG_O = KT * 32 * 4;
  static constexpr int L0F = KP * 4;
  static constexpr int BIASH = NH * NT * 8;
  static constexpr int NHP = (NH + 3) / 4 * 4;
  static constexpr int NET_WORDS = FRAG_H + FRAG_O + L0F + BIASH + 2 * NHP + 8;
};

template <int HID, int NL>
struct NetView {
  using C = MmaCfg<HID, NL>;
  uint32_t* fragH;
  uint32_t* fragO;
  float* l0;
  float* biasH;
  float* scaleH;
  int* modeH;
  float* biasO;
  __device__ explicit NetView(uint32_t* base) {
    fragH = base;
    fragO = fragH + C::FRAG_H;
    l0 = reinterpret_cast<float*>(fragO + C::FRAG_O);
    biasH = l0 + C::L0F;
    scaleH = biasH + C::BIASH;
    modeH = reinterpret_cast<int*>(scaleH + C::NHP);
    biasO = reinterpret_cast<float*>(modeH + C::NHP);
  }
  // B[k][n] entry of a fragment array with NTS n-tiles per k-tile.
  __device__ __forceinline__ static void put_b(uint32_t* frag, int nts, int k, int n, float hi, float lo) {
    const int t = k >> 4, kk = k & 15, j = n >> 3, g = n & 7;
    const int reg = kk >> 3, tq = (kk & 7) >> 1, half = kk & 1;
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(frag + ((t * nts + j) * 32 + g * 4 + tq) * 4);
    p[reg * 2 + half] = __float2bfloat16_rn(hi);
    p[(reg + 2) * 2 + half] = __float2bfloat16_rn(lo);
  }
  __device__ __forceinline__ static void put_b_split(uint32_t* frag, int nts, int k, int n, float v) {
    const float h = __bfloat162float(__float2bfloat16_rn(v));
    put_b(frag, nts, k, n, h, v - h);
  }
};

// Per-image coordinate tables (built in the prologue): colx[c], rowy[r] are
// the source coordinates of output column c / row r after crop / flip; NaN
// marks padding (AUG_OFFSET outside the source image).  rowy[out_h] repeats
// rowy[out_h - 1] (tables hold round4(W) + round4(H + 1) floats) so that a
// one-row look-ahead needs no clamp.
__device__ __forceinline__ void build_coord_tables(const DecodeArgs& a, const float* __restrict__ aug, int64_t img,
                                                   float* colx, float* rowy, int tid, int nthr) {
  const float nan = __int_as_float(0x7fc00000);
  float q[5] = {0.f, 0.f, 1.f, 1.f, 0.f};
  if (a.aug != RINR_AUG_NONE) {
#pragma unroll
    for (int i = 0; i < 5; ++i) q[i] = aug[img * 5 + i];
  }
  for (int i = tid; i <= a.out_w + a.out_h; i += nthr) {
    const bool is_col = i < a.out_w;
    const int n = is_col ? a.out_w : a.out_h;
    const double inv = is_col ? a.inv_wm1 : a.inv_hm1;
    const int slot = is_col ? i : i - a.out_w;
    const int k = slot < n ? slot : n - 1;
    float v;
    if (a.aug == RINR_AUG_NONE) {
      v = grid_coord(k, n, inv);
    } else if (a.aug == RINR_AUG_OFFSET) {
      const int s = (is_col ? ((int(q[2]) ? n - 1 - k : k) + int(q[0])) : k + int(q[1])) - int(q[3]);
      v = (s >= 0 && s < n) ? grid_coord(s, n, inv) : nan;
    } else {
      const int kk = (is_col && int(q[4])) ? n - 1 - k : k;
      v = is_col ? __fadd_rn(__fmul_rn(q[2], grid_coord(kk, n, inv)), q[0])
                 : __fadd_rn(__fmul_rn(q[3], grid_coord(kk, n, inv)), q[1]);
    }
    if (is_col) colx[k] = v;
    else rowy[slot] = v;
  }
}

// Affine (code - zero_point) of entry j, or 0 when pruned.
// B fragment word set of one lane for k-tile t, n-tile j of a layer (row-major
// (out, in) weights; B[k][n] = W[n][k]): {b0 hi, b1 hi, b0 lo, b1 lo}, b0 =
// (k = 16t+2tq, +1), b1 = (k + 8, k + 9), n = 8j + g; entries outside
// (fo, fi) are zero.  INT: integer codes (exact in bf16, lo = 0); else
// mul * value split into bf16 hi + lo (= NetView::put_b_split).
// SPREAD: output row o goes to column 2o (odd columns zero), so that the C
// fragment's first value of lane (g, tq) is output tq (persist.cuh epilogue).
template <bool INT, int KIND = VK_GEN, bool SPREAD = false>
__device__ __forceinline__ uint4 frag_words(const uint8_t* rec, const ValueRecipe& R, const WarpBits& B, int fi,
                                            int fo, int t, int j, float mul, int lane) {
  const int g = lane >> 2, tq = lane & 3, n = 8 * j + g;
  const int o = SPREAD ? n >> 1 : n;
  float v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = 16 * t + 2 * tq + (q & 1) + 8 * (q >> 1);
    const bool valid = k < fi && o < fo && !(SPREAD && (n & 1));
    const float x = value_at<INT, KIND>(rec, R, B, valid ? o * fi + k : 0);
    v[q] = valid ? (INT ? x : __fmul_rn(mul, x)) : 0.0f;
  }
  uint4 r;
  const __nv_bfloat162 h01 = __floats2bfloat162_rn(v[0], v[1]), h23 = __floats2bfloat162_rn(v[2], v[3]);
  r.x = bf2_bits(h01);
  r.y = bf2_bits(h23);
  r.z = bf2_bits(__floats2bfloat162_rn(v[0] - __low2float(h01), v[1] - __high2float(h01)));
  r.w = bf2_bits(__floats2bfloat162_rn(v[2] - __low2float(h23), v[3] - __high2float(h23)));
  return r;
}

__device__ __forceinline__ float dq_int(const uint8_t* rec, const DLayer& L, const uint32_t* words,
                                        const uint32_t* prefix, int j) {
  bool kept = true;
  int vi = j;
  if (L.form != FORM_DENSE) {
    const uint32_t wd = words[j >> 5];
    kept = (wd >> (j & 31)) & 1u;
    if (L.form == FORM_SPARSE) vi = int(prefix[j >> 5] + __popc(wd & ((1u << (j & 31)) - 1u)));
  }
  if (!kept) return 0.0f;
  const int code = int(rec[L.vals_off + vi]);
  return float(code - L.zp);
}

}  // namespace rinr
