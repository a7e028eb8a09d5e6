// Batched INR decode kernels for sm_100a.
//
//   dequantize_kernel   rinr_dequantize: materialised f32 parameters, bit-exact
//                       with reference archive.materialize (archive.py:278-325).
//   decode_generic      RINR_PREC_EXACT and any non-specialised architecture:
//                       fp32 FFMA on CUDA cores (reference net.py:183-214).
//   decode_mma<HID,NL>  uniform-width SIREN [2, HID x (NL-1), 3]: layer 0 on FFMA
//                       straight into the bf16 A-fragment layout, hidden layers
//                       as a register-resident mma.sync.m16n8k16 chain (the f32
//                       accumulator of two adjacent n8 tiles IS the A fragment
//                       of the next k16 tile, so sine -> bf16 pack -> next MMA
//                       never touches shared memory), bias preloaded into the
//                       accumulator, omega folded into the weights, MUFU sine,
//                       fused clamp/normalise epilogue through a per-warp
//                       shared-memory stage for coalesced stores.
// All kernels start with the same prologue: the record's bytes are copied
// from the HBM store to shared memory and dequantised there.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>
#include <string>
#include <unordered_map>

#include "device_common.cuh"

namespace rinr {

// ============================================================================
// rinr_dequantize
// ============================================================================
constexpr int kDqThreads = 128;

__global__ void __launch_bounds__(kDqThreads) dequantize_kernel(StoreView sv, const int64_t* __restrict__ ids,
                                                                int64_t n, float* __restrict__ out,
                                                                int64_t stride, int32_t* status) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t i = blockIdx.x;
  const int64_t id = ids[i];
  if (id < 0 || id >= sv.n) {
    if (threadIdx.x == 0) flag_bad_id(status, n, i);
    return;
  }
  uint8_t* rec = smem;
  const int nwords = (sv.max_width * sv.max_width + 31) / 32 + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + sv.max_record_bytes + 16);
  uint32_t* prefix = words + nwords;
  const uint32_t* lo = sv.lay_off + id * sv.lstride;
  const uint16_t* dims = sv.arch_dims + int(sv.arch_idx[id]) * kMaxDims;
  const int nl = sv.arch_nd[sv.arch_idx[id]] - 1;
  copy_record(rec, sv.blob + sv.rec_off[id], (lo[nl] + 15u) & ~15u, threadIdx.x, blockDim.x);
  __syncthreads();
  float* dst = out + i * stride;
  for (int l = 0; l < nl; ++l) {
    DLayer L = parse_layer(rec, lo[l], lo[l + 1], dims[l], dims[l + 1]);
    if (L.form != FORM_DENSE && threadIdx.x < 32) build_bit_prefix(rec, L, words, prefix, threadIdx.x);
    __syncthreads();
    for (int j = threadIdx.x; j < L.n; j += blockDim.x) dst[j] = dq_weight(rec, L, words, prefix, j);
    for (int o = threadIdx.x; o < L.out; o += blockDim.x) dst[L.n + o] = dq_bias(rec, L, o);
    dst += L.n + L.out;
    __syncthreads();
  }
}

// ============================================================================
// Generic fp32 decode (any architecture up to the store limits)
// ============================================================================
constexpr int kGenThreads = 128;

template <bool ACCURATE>
__global__ void __launch_bounds__(kGenThreads) decode_generic(StoreView sv, const int64_t* __restrict__ ids, int64_t n,
                                                              DecodeArgs a, const float* __restrict__ aug,
                                                              void* __restrict__ out, int32_t* status, int chunks) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t img = blockIdx.x / chunks;
  const int chunk = blockIdx.x % chunks;
  const int64_t id = ids[img];
  if (id < 0 || id >= sv.n) {
    if (threadIdx.x == 0 && chunk == 0) flag_bad_id(status, n, img);
    return;
  }
  const int tid = threadIdx.x;
  uint8_t* rec = smem;
  const int nwords = (sv.max_width * sv.max_width + 31) / 32 + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + sv.max_record_bytes + 16);
  uint32_t* prefix = words + nwords;
  float* wts = reinterpret_cast<float*>(prefix + nwords);
  float* act = wts + ((sv.max_params + 3) & ~3);  // [2][max_width][kGenThreads]

  const int ai = sv.arch_idx[id];
  const uint16_t* dims = sv.arch_dims + ai * kMaxDims;
  const int nl = sv.arch_nd[ai] - 1;
  const float omega = sv.arch_omega[ai];
  const uint32_t* lo = sv.lay_off + id * sv.lstride;
  copy_record(rec, sv.blob + sv.rec_off[id], (lo[nl] + 15u) & ~15u, tid, kGenThreads);
  __syncthreads();
  {
    float* dst = wts;
    for (int l = 0; l < nl; ++l) {
      DLayer L = parse_layer(rec, lo[l], lo[l + 1], dims[l], dims[l + 1]);
      if (L.form != FORM_DENSE && tid < 32) build_bit_prefix(rec, L, words, prefix, tid);
      __syncthreads();
      for (int j = tid; j < L.n; j += kGenThreads) dst[j] = dq_weight(rec, L, words, prefix, j);
      for (int o = tid; o < L.out; o += kGenThreads) dst[L.n + o] = dq_bias(rec, L, o);
      dst += L.n + L.out;
      __syncthreads();
    }
  }
  const int mw = sv.max_width;
  float* act0 = act;
  float* act1 = act + mw * kGenThreads;
  const int per = (a.hw + chunks - 1) / chunks;
  const int p0 = chunk * per, p1 = min(a.hw, p0 + per);
  for (int pb = p0; pb < p1; pb += kGenThreads) {
    const int p = pb + tid;
    if (p >= p1) break;
    float x, y;
    const bool valid = pixel_coord(a, aug, img, p, x, y);
    float* in = act0;
    float* nx = act1;
    in[0 * kGenThreads + tid] = x;
    in[1 * kGenThreads + tid] = y;
    const float* w = wts;
    float rgb[3] = {0.f, 0.f, 0.f};
    for (int l = 0; l < nl; ++l) {
      const int fi = dims[l], fo = dims[l + 1];
      const float* b = w + fi * fo;
      const bool last = l == nl - 1;
      for (int o = 0; o < fo; ++o) {
        const float* wr = w + o * fi;
        float z = 0.0f;
        for (int k = 0; k < fi; ++k) z = fmaf(in[k * kGenThreads + tid], wr[k], z);
        z = z + b[o];
        if (last) {
          rgb[o] = z;
        } else {
          const float arg = omega * z;
          nx[o * kGenThreads + tid] = ACCURATE ? sinf(arg) : __sinf(arg);
        }
      }
      w = b + fo;
      float* t = in;
      in = nx;
      nx = t;
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) store_value(a, out, img, p, ch, epilogue_value(a, rgb[ch], valid, ch));
  }
}

// ============================================================================
// Uniform-width SIREN on mma.sync.m16n8k16 (bf16 in, f32 accumulate)
// ============================================================================
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bf2_bits(__nv_bfloat162 v) { return *reinterpret_cast<uint32_t*>(&v); }

// (x0, x1) -> packed bf16x2 hi, and lo = bf16(x - f32(hi)) for the x3 split.
template <bool X3>
__device__ __forceinline__ void pack_act(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
  hi = bf2_bits(h);
  if constexpr (X3) {
    float2 hf = __bfloat1622float2(h);
    lo = bf2_bits(__floats2bfloat162_rn(x0 - hf.x, x1 - hf.y));
  }
}

template <bool ACCURATE>
__device__ __forceinline__ float sine(float x) {
  if constexpr (ACCURATE) return sinf(x);
  return __sinf(x);
}

// Shared-memory image of one record's decoded network (zero padded):
//   fragH[h][t][j][lane] : B fragments of hidden layer h+1, k-tile t, n-tile j
//                          X3: uint4 {b0 hi, b1 hi, b0 lo, b1 lo}; else uint2
//   fragO[t][lane]       : B fragments of the last layer (n-tile 0, 3 valid cols)
//   l0[c]                : float4 {omega*w[c][0], omega*w[c][1], omega*b[c], 0}
//   biasH[h][c]          : omega * b of hidden layer h+1;  biasO[8]
template <int HID, int NL, bool X3>
struct MmaCfg {
  static constexpr int KP = (HID + 15) / 16 * 16;
  static constexpr int KT = KP / 16;
  static constexpr int NT = (HID + 7) / 8;
  static constexpr int NH = NL - 2;
  static constexpr int FW = X3 ? 4 : 2;  // u32 words per lane per fragment
  static constexpr int FRAG_H = NH * KT * NT * 32 * FW;  // u32 words
  static constexpr int FRAG_O = KT * 32 * FW;
  static constexpr int L0F = KP * 4;                      // floats
  static constexpr int BIASH = NH * NT * 8;
  static constexpr int NET_WORDS = FRAG_H + FRAG_O + L0F + BIASH + 8;
};

template <int HID, int NL, bool X3>
struct NetSmem {
  using C = MmaCfg<HID, NL, X3>;
  uint32_t* fragH;
  uint32_t* fragO;
  float* l0;
  float* biasH;
  float* biasO;
  __device__ explicit NetSmem(uint32_t* base) {
    fragH = base;
    fragO = fragH + C::FRAG_H;
    l0 = reinterpret_cast<float*>(fragO + C::FRAG_O);
    biasH = l0 + C::L0F;
    biasO = biasH + C::BIASH;
  }
  // Place B[k][n] = value of the (k, n) entry of a hidden/last-layer operand.
  __device__ __forceinline__ void put_b(uint32_t* frag, int t_stride_words, int k, int n, float v) {
    const int t = k >> 4, kk = k & 15, j = n >> 3, g = n & 7;
    const int reg = kk >> 3, tq = (kk & 7) >> 1, half = kk & 1;
    const int lane = g * 4 + tq;
    __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(frag + ((t * t_stride_words + j) * 32 + lane) * C::FW);
    __nv_bfloat16 h = __float2bfloat16_rn(v);
    base[reg * 2 + half] = h;
    if constexpr (X3) base[(reg + 2) * 2 + half] = __float2bfloat16_rn(v - __bfloat162float(h));
  }
};

template <int HID, int NL, bool X3, bool ACCURATE, int WARPS, int NB>
__global__ void __launch_bounds__(WARPS * 32) decode_mma(StoreView sv, const int64_t* __restrict__ ids, int64_t n,
                                                         DecodeArgs a, const float* __restrict__ aug,
                                                         void* __restrict__ out, int32_t* status, int chunks,
                                                         float omega) {
  using C = MmaCfg<HID, NL, X3>;
  constexpr int NTHR = WARPS * 32;
  extern __shared__ __align__(16) uint8_t smem[];
  const int64_t img = blockIdx.x / chunks;
  const int chunk = blockIdx.x % chunks;
  const int64_t id = ids[img];
  if (id < 0 || id >= sv.n) {
    if (threadIdx.x == 0 && chunk == 0) flag_bad_id(status, n, img);
    return;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t* netw = reinterpret_cast<uint32_t*>(smem);
  NetSmem<HID, NL, X3> net(netw);
  // The record buffer is dead after the prologue; the epilogue stage reuses it.
  uint8_t* rec = smem + C::NET_WORDS * 4;
  constexpr int kWords = (HID * HID + 31) / 32 + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(rec + sv.max_record_bytes + 16);
  uint32_t* prefix = words + kWords;

  // ---- prologue: record -> smem, zero the padded operands, dequantise -----
  const uint32_t* lo = sv.lay_off + id * sv.lstride;
  copy_record(rec, sv.blob + sv.rec_off[id], (lo[NL] + 15u) & ~15u, tid, NTHR);
  for (int i = tid; i < C::NET_WORDS; i += NTHR) netw[i] = 0u;
  __syncthreads();
#pragma unroll 1
  for (int l = 0; l < NL; ++l) {
    const int fi = l == 0 ? 2 : HID, fo = l == NL - 1 ? 3 : HID;
    DLayer L = parse_layer(rec, lo[l], lo[l + 1], fi, fo);
    if (L.form != FORM_DENSE && warp == 0) build_bit_prefix(rec, L, words, prefix, lane);
    __syncthreads();
    for (int j = tid; j < L.n; j += NTHR) {
      const float w = dq_weight(rec, L, words, prefix, j);
      const int o = j / fi, k = j - o * fi;
      if (l == 0) {
        net.l0[o * 4 + k] = __fmul_rn(omega, w);
      } else if (l < NL - 1) {
        net.put_b(net.fragH + (l - 1) * C::KT * C::NT * 32 * C::FW, C::NT, k, o, __fmul_rn(omega, w));
      } else {
        net.put_b(net.fragO, 1, k, o, w);
      }
    }
    for (int o = tid; o < fo; o += NTHR) {
      const float b = dq_bias(rec, L, o);
      if (l == 0) net.l0[o * 4 + 2] = __fmul_rn(omega, b);
      else if (l < NL - 1) net.biasH[(l - 1) * C::NT * 8 + o] = __fmul_rn(omega, b);
      else net.biasO[o] = b;
    }
    __syncthreads();
  }

  // ---- main loop: each warp takes NB 16-pixel blocks at a time -----------
  const int g = lane >> 2, tq = lane & 3;
  float* stage = reinterpret_cast<float*>(rec) + warp * (3 * NB * 16);
  const int nblk = (a.hw + 15) / 16;
  const int per = (nblk + chunks - 1) / chunks;
  const int b0 = chunk * per, b1 = min(nblk, b0 + per);

  // Last-layer operands stay in registers for the whole chunk.
  uint32_t bo[C::KT][C::FW];
#pragma unroll
  for (int t = 0; t < C::KT; ++t)
#pragma unroll
    for (int r = 0; r < C::FW; ++r) bo[t][r] = net.fragO[(t * 32 + lane) * C::FW + r];
  const float bias_o0 = net.biasO[2 * tq], bias_o1 = net.biasO[2 * tq + 1];

#pragma unroll 1
  for (int gb = b0 + warp * NB; gb < b1; gb += WARPS * NB) {
    // -- layer 0 (2 -> HID) on FFMA, written in A-fragment order ---------
    uint32_t ah[NB][C::KT][4], al[NB][C::KT][4];
    bool valid[NB][2];
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float xr[2], yr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = (gb + b) * 16 + g + 8 * h;
        if (p < a.hw) {
          valid[b][h] = pixel_coord(a, aug, img, p, xr[h], yr[h]);
        } else {
          valid[b][h] = false;
          xr[h] = yr[h] = 0.0f;
        }
      }
#pragma unroll
      for (int t = 0; t < C::KT; ++t) {
        float s[2][4];  // [row half][col slot]: cols 16t+2tq, +1, 16t+8+2tq, +1
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int col = 16 * t + 2 * tq + (q & 1) + 8 * (q >> 1);
          const float4 w = *reinterpret_cast<const float4*>(net.l0 + col * 4);
#pragma unroll
          for (int h = 0; h < 2; ++h)
            s[h][q] = col < HID ? sine<ACCURATE>(fmaf(w.y, yr[h], fmaf(w.x, xr[h], w.z))) : 0.0f;
        }
        pack_act<X3>(s[0][0], s[0][1], ah[b][t][0], al[b][t][0]);
        pack_act<X3>(s[1][0], s[1][1], ah[b][t][1], al[b][t][1]);
        pack_act<X3>(s[0][2], s[0][3], ah[b][t][2], al[b][t][2]);
        pack_act<X3>(s[1][2], s[1][3], ah[b][t][3], al[b][t][3]);
      }
    }
    // -- hidden layers: register-resident MMA chain -----------------------
#pragma unroll 1
    for (int hl = 0; hl < C::NH; ++hl) {
      const uint32_t* fr = net.fragH + hl * C::KT * C::NT * 32 * C::FW;
      const float* bh = net.biasH + hl * C::NT * 8;
      float acc[NB][C::NT][4];
#pragma unroll
      for (int j = 0; j < C::NT; ++j) {
        const float2 bb = *reinterpret_cast<const float2*>(bh + 8 * j + 2 * tq);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          acc[b][j][0] = bb.x;
          acc[b][j][1] = bb.y;
          acc[b][j][2] = bb.x;
          acc[b][j][3] = bb.y;
        }
      }
#pragma unroll
      for (int t = 0; t < C::KT; ++t) {
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          const uint32_t* f = fr + ((t * C::NT + j) * 32 + lane) * C::FW;
          uint32_t bf[C::FW];
          if constexpr (X3) {
            const uint4 v = *reinterpret_cast<const uint4*>(f);
            bf[0] = v.x; bf[1] = v.y; bf[2] = v.z; bf[3] = v.w;
          } else {
            const uint2 v = *reinterpret_cast<const uint2*>(f);
            bf[0] = v.x; bf[1] = v.y;
          }
#pragma unroll
          for (int b = 0; b < NB; ++b) {
            if constexpr (X3) {
              mma16816(acc[b][j], al[b][t], bf[0], bf[1]);
              mma16816(acc[b][j], ah[b][t], bf[2], bf[3]);
            }
            mma16816(acc[b][j], ah[b][t], bf[0], bf[1]);
          }
        }
      }
      // sine -> next A fragments (n-tiles 2t, 2t+1 -> k-tile t)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
#pragma unroll
        for (int t = 0; t < C::KT; ++t) {
          float s[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int j = 2 * t + (e >> 2);
            s[e] = j < C::NT ? sine<ACCURATE>(acc[b][j < C::NT ? j : 0][e & 3]) : 0.0f;
          }
          pack_act<X3>(s[0], s[1], ah[b][t][0], al[b][t][0]);
          pack_act<X3>(s[2], s[3], ah[b][t][1], al[b][t][1]);
          pack_act<X3>(s[4], s[5], ah[b][t][2], al[b][t][2]);
          pack_act<X3>(s[6], s[7], ah[b][t][3], al[b][t][3]);
        }
      }
    }
    // -- last layer (HID -> 3) + epilogue ---------------------------------
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      float o[4] = {bias_o0, bias_o1, bias_o0, bias_o1};
#pragma unroll
      for (int t = 0; t < C::KT; ++t) {
        if constexpr (X3) {
          mma16816(o, al[b][t], bo[t][0], bo[t][1]);
          mma16816(o, ah[b][t], bo[t][2], bo[t][3]);
        }
        mma16816(o, ah[b][t], bo[t][0], bo[t][1]);
      }
      // o[0]=(px g, ch 2tq) o[1]=(g, 2tq+1) o[2]=(g+8, 2tq) o[3]=(g+8, 2tq+1)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ch = 2 * tq + (e & 1);
        const int row = g + 8 * (e >> 1);
        if (ch < 3) stage[ch * (NB * 16) + b * 16 + row] = epilogue_value(a, o[e], valid[b][e >> 1], ch);
      }
    }
    __syncwarp();
    const int pbase = gb * 16;
    if (a.layout == RINR_LAYOUT_NCHW) {
#pragma unroll
      for (int i = lane; i < 3 * NB * 16; i += 32) {
        const int ch = i / (NB * 16), q = i - ch * (NB * 16);
        const int p = pbase + q;
        if (p < a.hw && gb + q / 16 < b1) store_value(a, out, img, p, ch, stage[i]);
      }
    } else {
#pragma unroll
      for (int i = lane; i < 3 * NB * 16; i += 32) {
        const int q = i / 3, ch = i - q * 3;
        const int p = pbase + q;
        if (p < a.hw && gb + q / 16 < b1) store_value(a, out, img, p, ch, stage[ch * (NB * 16) + q]);
      }
    }
    __syncwarp();
  }
}

// ============================================================================
// Launchers
// ============================================================================
static int num_sms() {
  static int sms = [] {
    int d = 0, v = 148;
    if (cudaGetDevice(&d) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    return v;
  }();
  return sms;
}

static int launch_fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  return set_error(RINR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Raise a kernel's dynamic shared-memory limit once (not per launch), so that
// launches stay legal inside CUDA-graph stream capture.
template <class K>
static bool ensure_smem(K kern, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> done;
  if (bytes <= 48 * 1024) return true;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(reinterpret_cast<const void*>(kern));
  if (it != done.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) != cudaSuccess) return false;
  done[reinterpret_cast<const void*>(kern)] = bytes;
  return true;
}

static size_t prefix_bytes(const StoreView& sv) {
  const int nwords = (sv.max_width * sv.max_width + 31) / 32 + 1;
  return size_t(2) * nwords * 4;
}

}  // namespace rinr

using namespace rinr;

int rinr_launch_dequantize(const StoreView& sv, const int64_t* d_ids, int64_t n, float* d_out, int64_t out_stride,
                           int32_t* d_status, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d_status && cudaMemsetAsync(d_status, 0, sizeof(int32_t), st) != cudaSuccess)
    return launch_fail("status reset");
  if (n > 0x7FFFFFFF) return set_error(RINR_ERR_INVALID_INPUT, "too many ids in one call");
  size_t smem = sv.max_record_bytes + 16 + prefix_bytes(sv);
  if (!ensure_smem(dequantize_kernel, smem))
    return launch_fail("dequantize smem attribute");
  dequantize_kernel<<<unsigned(n), kDqThreads, smem, st>>>(sv, d_ids, n, d_out, out_stride, d_status);
  if (cudaPeekAtLastError() != cudaSuccess) return launch_fail("dequantize launch");
  return RINR_OK;
}

namespace {

DecodeArgs make_args(const rinr_decode_params_t* p) {
  DecodeArgs a{};
  a.out_h = p->out_h;
  a.out_w = p->out_w;
  a.hw = p->out_h * p->out_w;
  a.inv_wm1 = p->out_w > 1 ? 1.0 / double(p->out_w - 1) : 0.0;
  a.inv_hm1 = p->out_h > 1 ? 1.0 / double(p->out_h - 1) : 0.0;
  a.dtype = p->out_dtype;
  a.layout = p->out_layout;
  a.aug = p->aug_mode;
  a.identity = 1;
  for (int c = 0; c < 3; ++c) {
    a.mean[c] = p->mean[c];
    a.stdv[c] = p->std[c];
    if (p->mean[c] != 0.0f || p->std[c] != 1.0f) a.identity = 0;
  }
  return a;
}

// Images are split into `chunks` pixel ranges so that the grid covers the
// 148 SMs at least ~4 CTAs deep even for small batches of large images.
int pick_chunks(int64_t n, int hw, int px_per_cta_min) {
  const int64_t target = int64_t(num_sms()) * 8;
  int chunks = 1;
  while (n * chunks < target && hw / (chunks * 2) >= px_per_cta_min) chunks *= 2;
  return chunks;
}

template <int HID, int NL, bool X3, bool ACC>
int launch_mma_t(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
                 int32_t* status, cudaStream_t st, float omega) {
  constexpr int WARPS = 4, NB = 2;
  using C = MmaCfg<HID, NL, X3>;
  const int chunks = pick_chunks(n, a.hw, WARPS * NB * 16 * 4);
  const size_t rec = size_t(sv.max_record_bytes) + 16 + prefix_bytes(sv);
  const size_t stage = size_t(WARPS) * 3 * NB * 16 * 4;
  const size_t smem = size_t(C::NET_WORDS) * 4 + (rec > stage ? rec : stage);
  auto kern = decode_mma<HID, NL, X3, ACC, WARPS, NB>;
  if (!ensure_smem(kern, smem)) return launch_fail("decode_mma smem attribute");
  const int64_t grid = n * chunks;
  if (grid > 0x7FFFFFFF) return set_error(RINR_ERR_INVALID_INPUT, "batch too large");
  kern<<<unsigned(grid), WARPS * 32, smem, st>>>(sv, ids, n, a, aug, out, status, chunks, omega);
  if (cudaPeekAtLastError() != cudaSuccess) return launch_fail("decode_mma launch");
  return RINR_OK;
}

template <int HID, int NL>
int launch_mma(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
               int32_t* status, cudaStream_t st, float omega, bool x3, bool acc) {
  if (x3) return acc ? launch_mma_t<HID, NL, true, true>(sv, ids, n, a, aug, out, status, st, omega)
                     : launch_mma_t<HID, NL, true, false>(sv, ids, n, a, aug, out, status, st, omega);
  return acc ? launch_mma_t<HID, NL, false, true>(sv, ids, n, a, aug, out, status, st, omega)
             : launch_mma_t<HID, NL, false, false>(sv, ids, n, a, aug, out, status, st, omega);
}

bool uniform_width(const HostArch& h, int hid, int nl) {
  if (h.nd != nl + 1 || h.dims[0] != 2 || h.dims[nl] != 3) return false;
  for (int i = 1; i < nl; ++i)
    if (h.dims[i] != hid) return false;
  return true;
}

}  // namespace

int rinr_launch_decode(const StoreView& sv, const HostArch* ua, const int64_t* d_ids, int64_t n,
                       const rinr_decode_params_t* p, const float* d_aug, void* d_out, int32_t* d_status,
                       void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d_status && cudaMemsetAsync(d_status, 0, sizeof(int32_t), st) != cudaSuccess) return launch_fail("status reset");
  const DecodeArgs a = make_args(p);
  if (a.dtype == RINR_OUT_U8 && !a.identity)
    return set_error(RINR_ERR_INVALID_INPUT, "u8 output takes no mean/std normalisation");
  const bool acc = p->sin_mode == RINR_SIN_ACCURATE;
  if (ua && p->precision != RINR_PREC_EXACT) {
    const bool x3 = p->precision == RINR_PREC_FP32;
    const float om = float(ua->omega);
    if (uniform_width(*ua, 15, 3)) return launch_mma<15, 3>(sv, d_ids, n, a, d_aug, d_out, d_status, st, om, x3, acc);
    if (uniform_width(*ua, 40, 10)) return launch_mma<40, 10>(sv, d_ids, n, a, d_aug, d_out, d_status, st, om, x3, acc);
    if (uniform_width(*ua, 32, 10)) return launch_mma<32, 10>(sv, d_ids, n, a, d_aug, d_out, d_status, st, om, x3, acc);
  }
  // Generic fp32 path: weights + per-thread activations in shared memory.
  const size_t smem = size_t(sv.max_record_bytes) + 16 + prefix_bytes(sv) + size_t((sv.max_params + 3) & ~3) * 4 +
                      size_t(2) * sv.max_width * kGenThreads * 4;
  if (smem > 227 * 1024)
    return set_error(RINR_ERR_UNSUPPORTED, "architecture too large for the generic decode kernel (" +
                                               std::to_string(smem) + " B of shared memory)");
  const int chunks = pick_chunks(n, a.hw, kGenThreads * 2);
  const int64_t grid = n * chunks;
  if (grid > 0x7FFFFFFF) return set_error(RINR_ERR_INVALID_INPUT, "batch too large");
  auto kern = acc ? decode_generic<true> : decode_generic<false>;
  if (!ensure_smem(kern, smem)) return launch_fail("decode_generic smem attribute");
  kern<<<unsigned(grid), kGenThreads, smem, st>>>(sv, d_ids, n, a, d_aug, d_out, d_status, chunks);
  if (cudaPeekAtLastError() != cudaSuccess) return launch_fail("decode_generic launch");
  return RINR_OK;
}
