// Device helpers shared by every kernel: unaligned reads of record bytes held
// in shared memory, the per-layer section walk, the bit-exact integer
// dequantisation (reference archive.py:278-325), coordinates
// (net.py:138-149) and the fused epilogue (clamp / pad fill / normalise /
// convert / store).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "rinr_internal.h"

namespace rinr {

// Checked builds (-DRINR_CHECKED, tools/checked_build.sh): bounds of every
// shared-memory access made through the helpers below, of record reads and of
// output stores are asserted on the device (compute-sanitizer is not
// available on the GPU pool).  Product builds compile the checks away.
#ifdef RINR_CHECKED
#define RINR_DCHECK(c)                                                              \
  do {                                                                              \
    if (!(c)) {                                                                     \
      printf("RINR_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__, \
             int(blockIdx.x), int(threadIdx.x), #c);                                \
      __trap();                                                                     \
    }                                                                               \
  } while (0)
#else
#define RINR_DCHECK(c) \
  do {                 \
  } while (0)
#endif

// [p, p + bytes) lies inside this CTA's shared memory window: past the
// reserved system region and below the end of the CTA's allocation
// (%aggr_smem_size counts the reserved region too)
__device__ __forceinline__ bool in_smem(const void* p, uint32_t bytes) {
  uint32_t aggr, rsv_end;
  asm("mov.u32 %0, %%aggr_smem_size;" : "=r"(aggr));
  asm("mov.u32 %0, %%reserved_smem_offset_end;" : "=r"(rsv_end));
  const uint64_t off = __cvta_generic_to_shared(p);
  return __isShared(p) && off >= rsv_end && off + bytes <= aggr;
}

// ---------------------------------------------------------------------------
// Byte access into a 16-B aligned shared-memory copy of a record.  Fields in
// the .rinr format are packed (no alignment), so 32-bit values are assembled
// from the two aligned words that cover them.  Buffers are over-allocated by
// 16 bytes so the second word is always in bounds.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_u32u(const uint8_t* base, uint32_t off) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(base + (off & ~3u));
  RINR_DCHECK(in_smem(w, 8));
  uint32_t lo = w[0], hi = w[1];
  return __funnelshift_r(lo, hi, (off & 3u) * 8u);
}
__device__ __forceinline__ uint32_t ld_u16u(const uint8_t* base, uint32_t off) { return ld_u32u(base, off) & 0xFFFFu; }
__device__ __forceinline__ double ld_f64u(const uint8_t* base, uint32_t off) {
  return __hiloint2double(int(ld_u32u(base, off + 4)), int(ld_u32u(base, off)));
}

// Copy `bytes` (multiple of 16, 16-B aligned source) from global to shared
// memory with 16-B vector loads spread over `nthr` threads.
__device__ __forceinline__ void copy_record(uint8_t* dst, const uint8_t* __restrict__ src, uint32_t bytes, int tid,
                                            int nthr) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (uint32_t i = tid; i < bytes / 16; i += nthr) d[i] = __ldg(s + i);
}

// One layer's sections, located from its tag offset and the next layer's
// offset (bias is the last 4*out bytes of the section; archive.py:112-137).
struct DLayer {
  int tag, form, cst;
  int in, out, n;
  double scale;
  int zp;
  uint32_t bits_off, vals_off, bias_off;
};

__device__ __forceinline__ DLayer parse_layer(const uint8_t* rec, uint32_t off, uint32_t next_off, int in, int out) {
  DLayer L;
  uint32_t h = ld_u32u(rec, off);
  L.tag = h & 0xFF;
  L.form = (h >> 8) & 0xFF;
  L.cst = (h >> 16) & 0xFF;
  L.in = in;
  L.out = out;
  L.n = in * out;
  uint32_t p = off + 3;
  L.scale = 1.0;
  L.zp = 0;
  if (L.tag == TAG_A8 || L.tag == TAG_A16) {
    L.scale = ld_f64u(rec, p);
    L.zp = int(ld_u32u(rec, p + 8));
    p += 12;
  }
  L.bits_off = p;
  if (L.form != FORM_DENSE) p += (uint32_t(L.n) + 7) / 8;
  L.vals_off = p;
  L.bias_off = next_off - 4u * uint32_t(out);
  return L;
}

// Word view of the kept-bitset (LSB-first, row-major; archive.py:122, 288-290)
// plus exclusive popcount prefix per word, so the value index of a sparse
// entry j is prefix[j/32] + popc(word[j/32] & ((1 << j%32) - 1)).  Built by
// one warp; caller synchronises before use.
__device__ __forceinline__ void build_bit_prefix(const uint8_t* rec, const DLayer& L, uint32_t* words,
                                                 uint32_t* prefix, int lane) {
  const int nw = (L.n + 31) / 32;
  uint32_t carry = 0;
  for (int base = 0; base < nw; base += 32) {
    int w = base + lane;
    uint32_t v = 0;
    if (w < nw) {
      v = ld_u32u(rec, L.bits_off + 4u * uint32_t(w));
      int rem = L.n - 32 * w;
      if (rem < 32) v &= (1u << rem) - 1u;  // bytes past the bitset belong to the values
      words[w] = v;
    }
    uint32_t c = __popc(v), incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (w < nw) prefix[w] = carry + incl - c;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// Materialised weight entry j (row-major (out, in)) of layer L — bit-exact
// with archive.materialize:
//   affine, not const : kept ? f32(f64(scale) * (f64(code) - f64(zp))) : +0.0
//   f32 / f16 / const : sparse ? (kept ? value : +0.0) : stored value
// Value of a weight entry whose kept bit / value index are known.
__device__ __forceinline__ float dq_value(const uint8_t* rec, const DLayer& L, bool kept, int vi) {
  const bool affine = L.tag == TAG_A8 || L.tag == TAG_A16;
  if (affine && !L.cst) {
    if (!kept) return 0.0f;
    uint32_t code = L.tag == TAG_A8 ? uint32_t(rec[L.vals_off + vi]) : ld_u16u(rec, L.vals_off + 2u * vi);
    double diff = double(code) - double(L.zp);  // exact: both are integers < 2^33
    return __double2float_rn(__dmul_rn(L.scale, diff));
  }
  if (L.form == FORM_SPARSE && !kept) return 0.0f;
  if (L.tag == TAG_F16) return __half2float(__ushort_as_half((unsigned short)ld_u16u(rec, L.vals_off + 2u * vi)));
  return __uint_as_float(ld_u32u(rec, L.vals_off + 4u * vi));
}

__device__ __forceinline__ float dq_weight(const uint8_t* rec, const DLayer& L, const uint32_t* words,
                                           const uint32_t* prefix, int j) {
  bool kept = true;
  int vi = j;
  if (L.form != FORM_DENSE) {
    uint32_t wd = words[j >> 5];
    kept = (wd >> (j & 31)) & 1u;
    if (L.form == FORM_SPARSE) vi = int(prefix[j >> 5] + __popc(wd & ((1u << (j & 31)) - 1u)));
  }
  return dq_value(rec, L, kept, vi);
}

// Register-resident kept-bitset of a layer with at most 1024 entries: lane i
// holds word i (bits past n cleared) and the popcount of words [0, i), so a
// lookup is two shuffles instead of a shared-memory table.  A dense layer
// reads as all-kept with prefix 32 i, so one branch-free lookup serves all
// three forms.
struct WarpBits {
  uint32_t w, p;
};

__device__ __forceinline__ WarpBits warp_bits(const uint8_t* rec, const DLayer& L, int lane) {
  if (L.form == FORM_DENSE) return WarpBits{0xffffffffu, 32u * uint32_t(lane)};
  const int nw = (L.n + 31) / 32;
  uint32_t v = 0;
  if (lane < nw) {
    v = ld_u32u(rec, L.bits_off + 4u * uint32_t(lane));
    const int rem = L.n - 32 * lane;
    if (rem < 32) v &= (1u << rem) - 1u;  // bytes past the bitset belong to the values
  }
  const uint32_t c = __popc(v);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  return WarpBits{v, incl - c};
}

// Warp-uniform decode recipe of one layer's values (dq_value without branches).
struct ValueRecipe {
  uint32_t vals_off, emask;
  int esize, zp;
  bool sparse, affine, f16, zero_unkept;
  double scale;
};

__device__ __forceinline__ ValueRecipe value_recipe(const DLayer& L) {
  ValueRecipe r;
  r.vals_off = L.vals_off;
  r.sparse = L.form == FORM_SPARSE;
  const bool aff_tag = L.tag == TAG_A8 || L.tag == TAG_A16;
  r.affine = aff_tag && !L.cst;  // const affine layers store exact f32 values
  r.f16 = L.tag == TAG_F16;
  r.esize = r.affine ? (L.tag == TAG_A8 ? 1 : 2) : (r.f16 ? 2 : 4);
  r.emask = r.esize == 1 ? 0xFFu : (r.esize == 2 ? 0xFFFFu : 0xFFFFFFFFu);
  r.zero_unkept = r.affine || r.sparse;
  r.zp = L.zp;
  r.scale = L.scale;
  return r;
}

// Storage kinds with a dedicated straight-line decode (value_at<..., KIND>).
enum ValueKind { VK_GEN = 0, VK_A8 = 1, VK_F32 = 2 };

__device__ __forceinline__ int value_kind(const DLayer& L) {
  const bool aff_tag = L.tag == TAG_A8 || L.tag == TAG_A16;
  if (L.tag == TAG_A8 && !L.cst) return VK_A8;
  if (L.tag == TAG_F32 || (aff_tag && L.cst)) return VK_F32;  // const affine layers store exact f32
  return VK_GEN;
}

// Entry j of the layer (every lane of the warp must call: shuffles).  INT:
// the integer code - zero_point of an affine8 layer (exact in bf16).
template <bool INT, int KIND = VK_GEN>
__device__ __forceinline__ float value_at(const uint8_t* rec, const ValueRecipe& R, const WarpBits& B, int j) {
  const uint32_t wd = __shfl_sync(0xffffffffu, B.w, j >> 5);
  const uint32_t pre = __shfl_sync(0xffffffffu, B.p, j >> 5);
  const uint32_t bit = uint32_t(j) & 31u;
  const bool kept = (wd >> bit) & 1u;
  const uint32_t vi = R.sparse ? pre + __popc(wd & ((1u << bit) - 1u)) : uint32_t(j);
  RINR_DCHECK(in_smem(rec + R.vals_off + vi * uint32_t(R.esize), 1));
  if constexpr (INT) {
    const int code = int(rec[R.vals_off + vi]);
    return kept ? float(code - R.zp) : 0.0f;
  } else if constexpr (KIND == VK_A8) {
    const uint32_t code = rec[R.vals_off + vi];
    const float x = __double2float_rn(__dmul_rn(R.scale, double(code) - double(R.zp)));
    return kept ? x : 0.0f;
  } else if constexpr (KIND == VK_F32) {
    const float x = __uint_as_float(ld_u32u(rec, R.vals_off + 4u * vi));
    return (R.sparse && !kept) ? 0.0f : x;
  } else {
    const uint32_t raw = ld_u32u(rec, R.vals_off + vi * uint32_t(R.esize));
    const uint32_t code = raw & R.emask;
    float x;
    if (R.affine) x = __double2float_rn(__dmul_rn(R.scale, double(code) - double(R.zp)));
    else x = R.f16 ? __half2float(__ushort_as_half((unsigned short)code)) : __uint_as_float(raw);
    return (R.zero_unkept && !kept) ? 0.0f : x;
  }
}

// An affine8 hidden layer may feed the MMA as integer B = code - zero_point
// (exact in bf16) only when every such difference is an integer of magnitude
// <= 256: codes are 0..255, so zero_point must lie in [-1, 256].  The
// reference quantizer gives zero points outside that range when all kept
// weights share one sign (compressor.py:175-185); those layers take the
// float hi/lo path instead.
__device__ __forceinline__ bool int_b_exact(const DLayer& L) {
  return L.tag == TAG_A8 && !L.cst && L.zp >= -1 && L.zp <= 256;
}

__device__ __forceinline__ float dq_bias(const uint8_t* rec, const DLayer& L, int o) {
  return __uint_as_float(ld_u32u(rec, L.bias_off + 4u * o));
}

// ---------------------------------------------------------------------------
// Coordinates: x = f32(f64(c) * (1.0 / (w-1))), last = 1.0, 1-px axis = 0
// (np.linspace + astype(f32), net.py:146-149).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float grid_coord(int i, int n, double inv) {
  if (n <= 1) return 0.0f;
  if (i == n - 1) return 1.0f;
  return __double2float_rn(double(i) * inv);
}

struct DecodeArgs {
  int out_h, out_w, hw;
  int64_t out_elems;      // n * 3 * hw: bound of every output index (checked builds)
  double inv_wm1, inv_hm1;
  int dtype, layout, aug;
  int identity;           // mean 0 / std 1: skip the normalise arithmetic
  float mean[3], stdv[3];
};

// Source coordinate of output pixel p of image `img` after the crop / flip
// transform (oracle: augment_coords).  Returns false for padding pixels.
__device__ __forceinline__ bool pixel_coord(const DecodeArgs& a, const float* __restrict__ aug, int64_t img, int p,
                                            float& x, float& y) {
  const int r = p / a.out_w;
  const int c = p - r * a.out_w;
  if (a.aug == RINR_AUG_NONE) {
    x = grid_coord(c, a.out_w, a.inv_wm1);
    y = grid_coord(r, a.out_h, a.inv_hm1);
    return true;
  }
  const float* q = aug + img * 5;
  if (a.aug == RINR_AUG_OFFSET) {
    const int dx = int(q[0]), dy = int(q[1]), flip = int(q[2]), pad = int(q[3]);
    const int sc = (flip ? a.out_w - 1 - c : c) + dx - pad;
    const int sr = r + dy - pad;
    const bool ok = sc >= 0 && sc < a.out_w && sr >= 0 && sr < a.out_h;
    x = ok ? grid_coord(sc, a.out_w, a.inv_wm1) : 0.0f;
    y = ok ? grid_coord(sr, a.out_h, a.inv_hm1) : 0.0f;
    return ok;
  }
  const int cx = int(q[4]) ? a.out_w - 1 - c : c;
  x = __fadd_rn(__fmul_rn(q[2], grid_coord(cx, a.out_w, a.inv_wm1)), q[0]);
  y = __fadd_rn(__fmul_rn(q[3], grid_coord(r, a.out_h, a.inv_hm1)), q[1]);
  return true;
}

// clamp [0,1] (decoder.py:35) -> zero-fill padding -> (v - mean) / std.
__device__ __forceinline__ float epilogue_value(const DecodeArgs& a, float raw, bool valid, int ch) {
  float v = fminf(fmaxf(raw, 0.0f), 1.0f);
  if (!valid) v = 0.0f;
  if (!a.identity) {
    // select, not index: a runtime index into the kernel-parameter array would
    // force a local-memory copy of DecodeArgs
    const float m = ch == 0 ? a.mean[0] : (ch == 1 ? a.mean[1] : a.mean[2]);
    const float s = ch == 0 ? a.stdv[0] : (ch == 1 ? a.stdv[1] : a.stdv[2]);
    v = __fdiv_rn(__fsub_rn(v, m), s);
  }
  return v;
}

// Store one channel value of pixel p of image img.
__device__ __forceinline__ void store_value(const DecodeArgs& a, void* __restrict__ out, int64_t img, int p, int ch,
                                            float v) {
  const int64_t idx = a.layout == RINR_LAYOUT_NCHW ? (img * 3 + ch) * int64_t(a.hw) + p
                                                   : (img * int64_t(a.hw) + p) * 3 + ch;
  RINR_DCHECK(idx >= 0 && idx < a.out_elems && p >= 0 && p < a.hw && ch >= 0 && ch < 3);
  if (a.dtype == RINR_OUT_F32) {
    static_cast<float*>(out)[idx] = v;
  } else if (a.dtype == RINR_OUT_BF16) {
    static_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(v);
  } else {
    // floor(v * 255 + 0.5) in f32 (image.py:55, bench.py:67)
    static_cast<uint8_t*>(out)[idx] = uint8_t(floorf(__fadd_rn(__fmul_rn(v, 255.0f), 0.5f)));
  }
}

__device__ __forceinline__ void flag_bad_id(int32_t* status, int64_t n, int64_t i) {
  if (status) atomicMax(status, int32_t(n - i));
}

}  // namespace rinr
