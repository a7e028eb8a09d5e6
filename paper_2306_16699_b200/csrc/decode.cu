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

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>

#include "device_common.cuh"
#include "persist.cuh"
#include "tc_decode.cuh"

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
  uint8_t* slot = smem;
  const int nwords = (sv.max_width * sv.max_width + 31) / 32 + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + sv.max_slot_bytes + 16);
  uint32_t* prefix = words + nwords;
  const uint16_t* dims = sv.arch_dims + int(sv.arch_idx[id]) * kMaxDims;
  const int nl = sv.arch_nd[sv.arch_idx[id]] - 1;
  uint64_t off;
  uint32_t bytes;
  slot_of(sv, id, off, bytes);
  copy_record(slot, sv.blob + off, bytes, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint32_t* lo = reinterpret_cast<const uint32_t*>(slot);
  const uint8_t* rec = slot + sv.hdr_bytes;
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
  uint8_t* slot = smem;
  const int nwords = (sv.max_width * sv.max_width + 31) / 32 + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(smem + sv.max_slot_bytes + 16);
  uint32_t* prefix = words + nwords;
  float* wts = reinterpret_cast<float*>(prefix + nwords);
  float* act = wts + ((sv.max_params + 3) & ~3);  // [2][max_width][kGenThreads]

  const int ai = sv.arch_idx[id];
  const uint16_t* dims = sv.arch_dims + ai * kMaxDims;
  const int nl = sv.arch_nd[ai] - 1;
  const float omega = sv.arch_omega[ai];
  uint64_t off;
  uint32_t bytes;
  slot_of(sv, id, off, bytes);
  copy_record(slot, sv.blob + off, bytes, tid, kGenThreads);
  __syncthreads();
  const uint32_t* lo = reinterpret_cast<const uint32_t*>(slot);
  const uint8_t* rec = slot + sv.hdr_bytes;
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
// Launchers
// ============================================================================
static int num_sms() {  // of the current device, cached per device
  static std::atomic<int> cache[64];
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return 148;
  int v = cache[d].load();
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d) != cudaSuccess || v <= 0) v = 148;
    cache[d].store(v);
  }
  return v;
}

static int launch_fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  return set_error(RINR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Raise a kernel's dynamic shared-memory limit once per device (not per
// launch), so that launches stay legal inside CUDA-graph stream capture.  The
// attribute belongs to the device's context, hence the (device, kernel) key.
template <class K>
static bool ensure_smem(K kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  if (bytes <= 48 * 1024) return true;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  const auto key = std::make_pair(dev, reinterpret_cast<const void*>(kern));
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) != cudaSuccess) return false;
  done[key] = bytes;
  return true;
}

static size_t prefix_bytes(const StoreView& sv) {
  const int nwords = (sv.max_width * sv.max_width + 31) / 32 + 1;
  return size_t(2) * nwords * 4;
}

}  // namespace rinr

using namespace rinr;

#ifdef RINR_DEV_KNOBS
// Development builds: the decode_persist timeline ([4][512][8] u64 ns) and
// dequant task durations ([512][16][2] u64).
extern "C" RINR_API int rinr_dev_times(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_dev_t, sizeof(g_dev_t)) == cudaSuccess ? RINR_OK : RINR_ERR_CUDA;
}
extern "C" RINR_API int rinr_dev_task_times(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_dev_task, sizeof(g_dev_task)) == cudaSuccess ? RINR_OK : RINR_ERR_CUDA;
}
extern "C" RINR_API int rinr_dev_tc_times(long long* host) {
  return cudaMemcpyFromSymbol(host, g_dev_tc, sizeof(g_dev_tc)) == cudaSuccess ? RINR_OK : RINR_ERR_CUDA;
}
#endif

int rinr_launch_dequantize(const StoreView& sv, const int64_t* d_ids, int64_t n, float* d_out, int64_t out_stride,
                           int32_t* d_status, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (d_status && cudaMemsetAsync(d_status, 0, sizeof(int32_t), st) != cudaSuccess)
    return launch_fail("status reset");
  if (n > 0x7FFFFFFF) return set_error(RINR_ERR_INVALID_INPUT, "too many ids in one call");
  size_t smem = sv.max_slot_bytes + 16 + prefix_bytes(sv);
  if (!ensure_smem(dequantize_kernel, smem))
    return launch_fail("dequantize smem attribute");
  dequantize_kernel<<<unsigned(n), kDqThreads, smem, st>>>(sv, d_ids, n, d_out, out_stride, d_status);
  if (cudaPeekAtLastError() != cudaSuccess) return launch_fail("dequantize launch");
  return RINR_OK;
}

namespace {

DecodeArgs make_args(const rinr_decode_params_t* p, int64_t n) {
  DecodeArgs a{};
  a.out_h = p->out_h;
  a.out_w = p->out_w;
  a.hw = p->out_h * p->out_w;
  a.out_elems = n * 3 * int64_t(a.hw);
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

template <int HID, int NL, bool X3, bool ACC, int NW, int NB, class M>
int launch_persist(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug,
                   void* out, int32_t* status, cudaStream_t st, float omega, int flags) {
  using C = MmaCfg<HID, NL>;
  constexpr int KW = (HID * HID + 31) / 32 + 1;
  PersistLayout lay{};
  lay.net_words = C::NET_WORDS;
  lay.tab_floats = ((a.out_w + 3) & ~3) + ((a.out_h + 4) & ~3);  // rowy[out_h]: look-ahead copy
  lay.rec_bytes = (sv.max_slot_bytes + 16 + 15) & ~15;
  lay.pfx_words = (NL * 2 * KW + 3) & ~3;
  const bool shared_tab = a.aug == RINR_AUG_NONE;
  const size_t fixed = size_t(NW) * (3 * NB * 16 + 64) * 4 + (shared_tab ? size_t(lay.tab_floats) * 4 : 0) + 64;
  const size_t per_img = size_t(lay.net_words) * 4 + size_t(lay.rec_bytes) + size_t(lay.pfx_words) * 4 + 16 +  // + metaid, ready
                         (shared_tab ? 0 : size_t(lay.tab_floats) * 4);
  constexpr int CPS = NW < 16 ? 16 / NW : 1;  // CTAs per SM
  const size_t budget = (228 * 1024) / CPS - 1024;
  if (fixed + per_img > budget) return set_error(RINR_ERR_UNSUPPORTED, "record or output too large for the decode kernel");
  const int sms = num_sms();
  const int64_t groups = n * ((((a.hw + 15) / 16) + NB - 1) / NB);
  if (groups >= (int64_t(1) << 31)) return set_error(RINR_ERR_INVALID_INPUT, "batch too large for one decode call");
  const int grid = int(groups < int64_t(CPS) * sms ? groups : int64_t(CPS) * sms);
  const int64_t imgs_per_cta = (n + grid - 1) / grid + 1;
  lay.maxi = int(std::min<int64_t>({int64_t((budget - fixed) / per_img), imgs_per_cta, 64}));
  const size_t smem = fixed + size_t(lay.maxi) * per_img;
  auto kern = decode_persist<HID, NL, X3, ACC, NW, NB, M>;
  if (!ensure_smem(kern, smem)) return launch_fail("decode_persist smem attribute");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // development knob for timing breakdowns, compiled only with -DRINR_DEV_KNOBS (it
  // produces wrong images): RINR_DEBUG_SKIP=1 skips phase 2, =2 the dequant, =3 both,
  // =4 everything after the CTA's work split (launch + PDL chain only)
#ifdef RINR_DEV_KNOBS
  static const int dbg = [] { const char* e = getenv("RINR_DEBUG_SKIP"); return e ? atoi(e) & 7 : 0; }();
#else
  constexpr int dbg = 0;
#endif
  int overlap = ((flags & RINR_FLAG_OVERLAP_PROLOGUE) ? 1 : 0) | (dbg << 1) |
                ((flags & RINR_FLAG_PREFETCH_NEXT) ? 64 : 0);
#ifdef RINR_DEV_KNOBS
  static std::atomic<int> dev_slot{0};
  overlap |= (dev_slot++ & 3) << 4;  // timeline slot of this launch (dev_stamp)
#endif
  if (cudaLaunchKernelEx(&cfg, kern, sv, ids, n, a, aug, out, status, omega, lay, overlap) != cudaSuccess)
    return launch_fail("decode_persist launch");

  return RINR_OK;
}

template <int HID, int NL, bool X3, bool ACC, int NW, int NB>
int launch_mode(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
                int32_t* status, cudaStream_t st, float omega, int flags) {
#define RINR_LAUNCH(AL, ST, IB) \
  launch_persist<HID, NL, X3, ACC, NW, NB, Mode<AL, ST, IB>>(sv, ids, n, a, aug, out, status, st, omega, flags)
#define RINR_LAUNCH_SEP(ST, IB) \
  launch_persist<HID, NL, X3, ACC, NW, NB, Mode<true, ST, IB, true>>(sv, ids, n, a, aug, out, status, st, omega, flags)
  constexpr int GPX = NB * 16;
  if constexpr (ACC) {
    return RINR_LAUNCH(false, 0, false);  // accurate-sine kernels: one generic store path
  } else {
    if (a.out_w % GPX != 0) return RINR_LAUNCH(false, 0, false);
    if constexpr (HID <= 16 && NB == 2) {
      // one 32-pixel row per group: separable layer 0 (one sine per row per
      // unit pair lane instead of one per pixel and unit)
      if (a.out_w == GPX) {
        const int st_mode = a.layout == RINR_LAYOUT_NCHW ? (a.dtype == RINR_OUT_F32 ? 1 : a.dtype == RINR_OUT_BF16 ? 2 : 0)
                                                          : (a.dtype == RINR_OUT_F32 ? 3 : 0);
        if (st_mode == 1) return sv.hidden_int8 ? RINR_LAUNCH_SEP(1, true) : RINR_LAUNCH_SEP(1, false);
        if (st_mode == 2) return sv.hidden_int8 ? RINR_LAUNCH_SEP(2, true) : RINR_LAUNCH_SEP(2, false);
        if (st_mode == 3) return sv.hidden_int8 ? RINR_LAUNCH_SEP(3, true) : RINR_LAUNCH_SEP(3, false);
        return RINR_LAUNCH_SEP(0, false);  // u8 / other layouts: same pixels, scalar stores
      }
    }
    if (sv.hidden_int8) {  // store-wide: every hidden layer is affine8 codes
      if (a.layout == RINR_LAYOUT_NCHW && a.dtype == RINR_OUT_F32) return RINR_LAUNCH(true, 1, true);
      if (a.layout == RINR_LAYOUT_NCHW && a.dtype == RINR_OUT_BF16) return RINR_LAUNCH(true, 2, true);
      if (a.layout == RINR_LAYOUT_NHWC && a.dtype == RINR_OUT_F32) return RINR_LAUNCH(true, 3, true);
    }
    if (a.layout == RINR_LAYOUT_NCHW && a.dtype == RINR_OUT_F32) return RINR_LAUNCH(true, 1, false);
    if (a.layout == RINR_LAYOUT_NCHW && a.dtype == RINR_OUT_BF16) return RINR_LAUNCH(true, 2, false);
    if (a.layout == RINR_LAYOUT_NHWC && a.dtype == RINR_OUT_F32) return RINR_LAUNCH(true, 3, false);
    return RINR_LAUNCH(true, 0, false);
  }
#undef RINR_LAUNCH
#undef RINR_LAUNCH_SEP
}

template <int HID, int NL, bool X3, int T, bool INTB>
int launch_tc_t(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
                int32_t* status, cudaStream_t st, float omega, int flags) {
  using C = TcCfg<HID, NL, INTB>;
  constexpr int KW = (HID * HID + 31) / 32 + 1;
  TcLayout lay{};
  lay.net_bytes = (C::NET_BYTES + 127) & ~127;
  lay.tab_floats = ((a.out_w + 3) & ~3) + ((a.out_h + 4) & ~3);  // rowy[out_h]: look-ahead copy
  lay.rec_bytes = (sv.max_slot_bytes + 16 + 15) & ~15;
  lay.pfx_words = (NL * 2 * KW + 3) & ~3;
  constexpr int SLOT = C::slot_cols(X3);
  lay.tmem_cols = T * SLOT <= 128 ? 128 : (T * SLOT <= 256 ? 256 : 512);
  static_assert(T * SLOT <= 512, "TMEM holds 512 columns");
  const bool shared_tab = a.aug == RINR_AUG_NONE;
  const size_t budget = 227 * 1024;
  auto need = [&](int maxi, size_t& r0) {
    r0 = size_t(maxi) * (lay.rec_bytes + size_t(lay.pfx_words) * 4);
    r0 = std::max(r0, size_t(4 * T) * 96 * 4);  // phase-2 reuse: per-warp output stage
    r0 = (r0 + 1023) & ~size_t(1023);
    return r0 + size_t(maxi) * lay.net_bytes + size_t(shared_tab ? 1 : maxi) * lay.tab_floats * 4 + 2 * T * 8 + 16 +
           size_t(maxi) * 8 + 64;
  };
  const int sms = num_sms();
  const int64_t tiles = n * ((a.hw + 127) / 128);
  const int grid = int(tiles < sms ? tiles : sms);
  const int64_t imgs_per_cta = (n + grid - 1) / grid + 1;
  int maxi = int(std::min<int64_t>(imgs_per_cta, 8));
  size_t r0 = 0;
  while (maxi > 1 && need(maxi, r0) > budget) --maxi;
  const size_t smem = need(maxi, r0);
  if (smem > budget) return set_error(RINR_ERR_UNSUPPORTED, "record too large for the tensor-core decode kernel");
  lay.maxi = maxi;
  lay.region0 = int(r0);
  auto kern = decode_tc<HID, NL, X3, T, INTB>;
  if (!ensure_smem(kern, smem)) return launch_fail("decode_tc smem attribute");
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(4 * T * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int overlap = (flags & RINR_FLAG_OVERLAP_PROLOGUE) ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, sv, ids, n, a, aug, out, status, omega, lay, overlap) != cudaSuccess)
    return launch_fail("decode_tc launch");
  return RINR_OK;
}

// T = tile slots in flight (4 epilogue warps each); INTB = store-wide
// "hidden layers are affine8" (no B lo arrays, frees shared memory for slots).
template <int HID, int NL, bool X3>
int launch_tc(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
              int32_t* status, cudaStream_t st, float omega, int flags) {
  // bf16 slots are 96 TMEM columns: 5 in flight (20 warps); X3 slots 128: 4
  constexpr int T = X3 ? 5 : 6;
  if (sv.hidden_int8) return launch_tc_t<HID, NL, X3, T, true>(sv, ids, n, a, aug, out, status, st, omega, flags);
  return launch_tc_t<HID, NL, X3, T, false>(sv, ids, n, a, aug, out, status, st, omega, flags);
}

template <int HID, int NL, bool X3, bool ACC>
int launch_mma_t(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
                 int32_t* status, cudaStream_t st, float omega, int flags) {
  if constexpr (HID <= 16) {
    // CTA shape = warps x (16-pixel blocks per warp), two 8-warp CTAs per SM:
    // with the separable layer 0 this is 1.5% faster than one 16-warp CTA
    // (67.7 vs 66.7 M img/s on c2) and 0.9% faster than four 4-warp CTAs; round 1
    // measured 16 x 2 best for the direct layer 0 against (8,4) (16,1) (24,1)
    // (32,1) and 20 x 2 at 92 registers.  RINR_NW=16 selects one 16-warp CTA.
    static const int nw = [] {
      const char* e = std::getenv("RINR_NW");
      return e ? atoi(e) : 8;
    }();
    if (nw == 8) return launch_mode<HID, NL, X3, ACC, 8, 2>(sv, ids, n, a, aug, out, status, st, omega, flags);
    return launch_mode<HID, NL, X3, ACC, 16, 2>(sv, ids, n, a, aug, out, status, st, omega, flags);
  } else {
    if constexpr (!ACC) {
      // wide nets: tcgen05 + TMEM kernel (RINR_NO_TC=1 selects the mma.sync chain, for A/B comparison)
      static const bool no_tc = [] {
        const char* e = std::getenv("RINR_NO_TC");
        return e && e[0] == '1';
      }();
      if (!no_tc) return launch_tc<HID, NL, X3>(sv, ids, n, a, aug, out, status, st, omega, flags);
    }
    return launch_mode<HID, NL, X3, ACC, 16, 1>(sv, ids, n, a, aug, out, status, st, omega, flags);
  }
}

template <int HID, int NL>
int launch_mma(const StoreView& sv, const int64_t* ids, int64_t n, const DecodeArgs& a, const float* aug, void* out,
               int32_t* status, cudaStream_t st, float omega, bool x3, bool acc, int flags) {
  if (x3) return acc ? launch_mma_t<HID, NL, true, true>(sv, ids, n, a, aug, out, status, st, omega, flags)
                     : launch_mma_t<HID, NL, true, false>(sv, ids, n, a, aug, out, status, st, omega, flags);
  return acc ? launch_mma_t<HID, NL, false, true>(sv, ids, n, a, aug, out, status, st, omega, flags)
             : launch_mma_t<HID, NL, false, false>(sv, ids, n, a, aug, out, status, st, omega, flags);
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
  const DecodeArgs a = make_args(p, n);
  if (a.dtype == RINR_OUT_U8 && !a.identity)
    return set_error(RINR_ERR_INVALID_INPUT, "u8 output takes no mean/std normalisation");
  const bool acc = p->sin_mode == RINR_SIN_ACCURATE;
  if (ua && p->precision != RINR_PREC_EXACT && a.hw < (1 << 24)) {
    const bool x3 = p->precision == RINR_PREC_FP32;
    const float om = float(ua->omega);
    if (uniform_width(*ua, 15, 3)) return launch_mma<15, 3>(sv, d_ids, n, a, d_aug, d_out, d_status, st, om, x3, acc, p->flags);
    if (uniform_width(*ua, 40, 10)) return launch_mma<40, 10>(sv, d_ids, n, a, d_aug, d_out, d_status, st, om, x3, acc, p->flags);
    if (uniform_width(*ua, 32, 10)) return launch_mma<32, 10>(sv, d_ids, n, a, d_aug, d_out, d_status, st, om, x3, acc, p->flags);
  }
  // Generic fp32 path: weights + per-thread activations in shared memory.
  const size_t smem = size_t(sv.max_slot_bytes) + 16 + prefix_bytes(sv) + size_t((sv.max_params + 3) & ~3) * 4 +
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
