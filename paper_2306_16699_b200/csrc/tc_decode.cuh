// Wide-net batched decode on 5th-generation tensor cores (tcgen05 + TMEM).
//
// For the 10-layer nets of the paper ([2,40x9,3] Mini-ImageNet, [2,32x9,3]
// 102flowers) the hidden-layer contractions dominate the tensor
// work and the register-resident mma.sync chain is register- and HMMA-bound.
// Here each 128-pixel tile of an image is one UMMA M=128 row block:
//
//   * activations (A, bf16 hi + lo) live in tensor memory next to the
//     accumulator (tcgen05.st, two bf16 per 32-bit column, lane = pixel), and
//     the MMA reads them from there (.ts form), so shared-memory bandwidth is
//     spent only on the weights;
//   * weights (B, [N][K] K-major, hi + lo, or exact integer codes for affine8
//     layers) are dequantised per image by phase 1 straight into that layout;
//   * one thread of each tile slot issues that slot's tcgen05.mma (kind::f16,
//     bf16 x bf16 -> f32, A from TMEM, B from smem) into the slot's TMEM
//     accumulator and commits to the slot's mbarrier, so slots never wait on
//     each other (no central MMA warp);
//   * four epilogue warps per tile slot (one TMEM lane quarter each, thread =
//     pixel) tcgen05.ld the accumulator row, apply scale/bias, take the MUFU
//     sine, split to bf16 hi/lo and write the next layer's A row.
// T tile slots are in flight, so the tensor core works on one slot while the
// epilogue warps of the others evaluate sines.  The output layer (HID -> 3) is
// an N=16 UMMA; clamp/normalise/store happen in the epilogue threads.
#pragma once

#include "persist.cuh"

namespace rinr {
#ifdef RINR_DEV_KNOBS
// Development timeline of CTA 0 (tools/dev_tc_timeline.py): clock64 of each
// slot's issuing thread per (round, layer): [0] before the MMA wait, [1] after
// it, [2] after the slot barrier (next A complete, MMA about to be issued),
// [3] after the MMAs and the commit are issued.
__device__ long long g_dev_tc[8][8][12][4];
#define RINR_TC_STAMP(s, r, l, k)                                                        \
  do {                                                                                   \
    if (blockIdx.x == 0 && issuer && (r) < 8 && (l) < 12) g_dev_tc[s][r][l][k] = clock64(); \
  } while (0)
#else
#define RINR_TC_STAMP(s, r, l, k) \
  do {                            \
  } while (0)
#endif
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory matrix descriptor, K-major, no swizzle (canonical
// ((8,n),2):((1,SBO),LBO) in 16-byte units), Blackwell version field = 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// Instruction descriptor: bf16 A/B, f32 D, K-major A and B, M x N.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
  const uint32_t a = smem_u32(mbar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32 lanes x 32 bit, 8 / 16 / 32 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// Ties registers loaded by tcgen05.ld to a point after tcgen05.wait::ld (the
// compiler may otherwise schedule their first use before the wait).
__device__ __forceinline__ void pin8(float (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) asm volatile("" : "+f"(v[i]));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D (+)= A[tmem] * B[smem]^T
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Whole-warp forms: every lane passes the same (warp-uniform) operands and
// elect.sync picks the issuing lane inside the asm, so the compiler needs no
// per-thread waterfall around the uniform-datapath instruction.  Measured on
// B200 (tools/micro/umma_lat.cu): 6 chained M128 N48 K16 MMAs + commit issue
// in 739 cycles this way against 885 from one thread of a divergent branch.
__device__ __forceinline__ void mma_bf16_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_warp(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(mbar))
      : "memory");
}

__device__ __forceinline__ void bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Byte offset of element (row, k) in a K-major core-matrix layout with
// `chunks` 8-element K chunks per 8-row group.
__device__ __forceinline__ uint32_t kmaj_off(int row, int k, int chunks) {
  return uint32_t(((row >> 3) * chunks + (k >> 3)) * 128 + (row & 7) * 16 + (k & 7) * 2);
}

}  // namespace tc

template <int HID, int NL, bool INTB>
struct TcCfg {
  static constexpr int KP = (HID + 15) / 16 * 16;  // K of the hidden/output layers
  static constexpr int NP = KP;                    // N of the hidden layers (M=128 needs N % 16 == 0)
  static constexpr int NO = 16;                    // N of the output layer (3 valid)
  static constexpr int CH = KP / 8;                // 8-element K chunks per row
  static constexpr int KS = KP / 16;               // UMMA K steps per layer
  static constexpr int NH = NL - 2;
  // per-image network in smem (bytes)
  static constexpr int BH_BYTES = NP * KP * 2;     // one hidden-layer B matrix (bf16)
  static constexpr int BO_BYTES = NO * KP * 2;
  // INTB: every hidden layer is integer-coded (exact in bf16): no B lo arrays
  static constexpr int BHL_BYTES = INTB ? 0 : BH_BYTES;
  static constexpr int NET_BYTES = NH * (BH_BYTES + BHL_BYTES) + BO_BYTES * 2 + KP * 16 + NH * KP * 4 + 16 * 4 + NH * 8;
  // TMEM columns per tile slot: D (NP f32) at +0, A hi at +64, A lo at +96
  // (X3); bf16 mode has no A lo, so its slots are 96 columns and 5 fit.
  static constexpr int SLOT_COLS = 128;
  // packed: D (NP f32 columns) | A hi (KP/2) | A lo (KP/2, X3 only)
  static constexpr int slot_cols(bool x3) { return (NP + (x3 ? KP : KP / 2) + 15) / 16 * 16; }
  static constexpr int ahi_col(bool) { return NP; }
  static constexpr int alo_col() { return NP + KP / 2; }
};

// Per-image network view (K-major B matrices + scalars).
template <int HID, int NL, bool INTB>
struct TcNet {
  using C = TcCfg<HID, NL, INTB>;
  uint8_t* bh_hi;  // [NH][NP x KP]
  uint8_t* bh_lo;
  uint8_t* bo_hi;  // [NO x KP]
  uint8_t* bo_lo;
  float* l0;       // [KP] float4 {omega w0, omega w1, omega b, 0}
  float* biasH;    // [NH][KP]
  float* biasO;    // [16]
  float* scaleH;   // [NH]
  int* modeH;      // [NH]
  __device__ explicit TcNet(uint8_t* base) {
    bh_hi = base;
    bh_lo = bh_hi + C::NH * C::BH_BYTES;  // unused (aliases bo_hi) when INTB
    bo_hi = bh_lo + C::NH * C::BHL_BYTES;
    bo_lo = bo_hi + C::BO_BYTES;
    l0 = reinterpret_cast<float*>(bo_lo + C::BO_BYTES);
    biasH = l0 + C::KP * 4;
    biasO = biasH + C::NH * C::KP;
    scaleH = biasO + 16;
    modeH = reinterpret_cast<int*>(scaleH + C::NH);
  }
  __device__ __forceinline__ static void put(uint8_t* hi, uint8_t* lo, int n, int k, float vhi, float vlo) {
    const uint32_t off = tc::kmaj_off(n, k, C::CH);
    *reinterpret_cast<__nv_bfloat16*>(hi + off) = __float2bfloat16_rn(vhi);
    if (lo) *reinterpret_cast<__nv_bfloat16*>(lo + off) = __float2bfloat16_rn(vlo);
  }
  __device__ __forceinline__ static void put_split(uint8_t* hi, uint8_t* lo, int n, int k, float v) {
    const float h = __bfloat162float(__float2bfloat16_rn(v));
    put(hi, lo, n, k, h, v - h);
  }
};

struct TcLayout {
  int region0;    // bytes of the A-tile / phase-1 scratch region
  int maxi;       // images per chunk
  int net_bytes;  // per image (16-B multiple)
  int tab_floats; // coordinate table per image (or shared)
  int rec_bytes;  // phase-1 record slot per image
  int pfx_words;  // phase-1 prefix scratch per image
  int tmem_cols;  // allocated TMEM columns
};

// Split x into bf16 hi (truncation) + lo (rounded remainder) and pack pairs.
template <bool X3>
__device__ __forceinline__ void split8(const float (&x)[8], uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) pack_act<X3>(x[2 * i], x[2 * i + 1], h[i], l[i]);
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Issue layer l's MMAs for one tile slot (l < NL-2: hidden layer l+1,
// l == NL-2: output layer) and commit them to the slot's mbarrier.  Called by
// the slot's whole first warp (converged); one elected lane issues.
#ifdef RINR_TC_THREAD_ISSUE
constexpr bool kWarpIssue = false;
#else
constexpr bool kWarpIssue = true;
#endif
// Each layer is one accumulator chain committed to the slot's mbarrier.  With
// RINR_TC_SPLITN (development option) hidden layers are issued as two chains
// over the N halves (32 + 16 columns for N = 48), each committed to its own
// barrier (mbar[s], mbar[T + s]), so the epilogue could start on the first
// columns while the tensor core computes the rest: measured 9% slower (twice
// the MMA instructions, tools/micro/umma_lat.cu).
#ifdef RINR_TC_SPLITN
constexpr bool kSplitN = true;
#else
constexpr bool kSplitN = false;
#endif
template <int HID, int NL, bool INTB>
struct SplitN {
  using C = TcCfg<HID, NL, INTB>;
  static constexpr bool ON = kSplitN && C::NP > 16;
  static constexpr int NA = ON ? (C::NP / 16 + 1) / 2 * 16 : C::NP;  // columns of the first chain
};

template <int HID, int NL, bool X3, bool INTB>
__device__ __forceinline__ void issue_layer(const TcNet<HID, NL, INTB>& net, uint32_t d, int l, uint64_t* mb0,
                                            uint64_t* mb1) {
  using C = TcCfg<HID, NL, INTB>;
  using SN = SplitN<HID, NL, INTB>;
  const uint32_t ahi = d + C::ahi_col(X3), alo = d + C::alo_col();
  const bool outl = l == NL - 2;
  const uint32_t bhi = tc::smem_u32(outl ? net.bo_hi : net.bh_hi + l * C::BH_BYTES);
  const uint32_t blo = tc::smem_u32(outl ? net.bo_lo : net.bh_lo + l * C::BH_BYTES);
  const bool int_b = !outl && (INTB || net.modeH[l] != 0);
  constexpr uint32_t SBO = C::CH * 128, LBO = 128;
  // one accumulator chain: D columns [dcol, dcol + n), B rows from brow
  auto chain = [&](uint32_t dcol, uint32_t brow, uint32_t idesc) {
    const uint32_t boff = (brow / 8) * SBO;
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
      const uint32_t koff = boff + uint32_t(ks * 2 * 128);  // B: two 8-element chunks per K step
      const uint32_t acol = uint32_t(ks * 8);                // A: 16 bf16 = 8 TMEM columns per K step
      auto mma = [&](uint32_t a, uint64_t b, uint32_t acc) {
        if constexpr (kWarpIssue) tc::mma_bf16_ts_warp(d + dcol, a, b, idesc, acc);
        else tc::mma_bf16_ts(d + dcol, a, b, idesc, acc);
      };
      mma(ahi + acol, tc::make_desc(bhi + koff, LBO, SBO), ks > 0);
      if (X3) mma(alo + acol, tc::make_desc(bhi + koff, LBO, SBO), 1);
      if (!int_b) mma(ahi + acol, tc::make_desc(blo + koff, LBO, SBO), 1);
    }
  };
  auto commit = [&](uint64_t* mb) {
    if constexpr (kWarpIssue) tc::commit_warp(mb);
    else tc::commit(mb);
  };
  if (outl) {
    chain(0, 0, tc::make_idesc(128, C::NO));
    commit(mb0);
    if constexpr (SN::ON) commit(mb1);  // both barriers complete once per layer
  } else if constexpr (SN::ON) {
    chain(0, 0, tc::make_idesc(128, SN::NA));
    commit(mb0);
    chain(SN::NA, SN::NA, tc::make_idesc(128, C::NP - SN::NA));
    commit(mb1);
  } else {
    chain(0, 0, tc::make_idesc(128, C::NP));
    commit(mb0);
  }
}

template <int HID, int NL, bool X3, int T, bool INTB>
__global__ void __launch_bounds__(4 * T * 32, 1)
    decode_tc(StoreView sv, const int64_t* __restrict__ ids, int64_t n, DecodeArgs a,
              const float* __restrict__ aug, void* __restrict__ out, int32_t* status, float omega, TcLayout lay,
              int overlap) {
  using C = TcCfg<HID, NL, INTB>;
  using Net = TcNet<HID, NL, INTB>;
  constexpr int NW = 4 * T;                 // 4 warps (one TMEM lane quarter each) per tile slot
  constexpr int NT = NW * 32;
  constexpr int KW = (HID * HID + 31) / 32 + 1;

  if (!overlap) pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem[];
  // ---- shared memory map ------------------------------------------------------
  uint8_t* nets = smem + lay.region0;                                // [maxi] networks
  float* tabs = reinterpret_cast<float*>(nets + lay.maxi * lay.net_bytes);
  const bool shared_tab = a.aug == RINR_AUG_NONE;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tabs + (shared_tab ? 1 : lay.maxi) * lay.tab_floats);  // [2T]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 2 * T);
  int64_t* metaid = reinterpret_cast<int64_t*>(tmem_slot + 4);      // [maxi]
  uint8_t* recs = smem;  // phase-1 scratch
  uint32_t* pfx = reinterpret_cast<uint32_t*>(recs + size_t(lay.maxi) * lay.rec_bytes);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ntile = (a.hw + 127) / 128;  // tiles per image
  const int64_t total = n * ntile;
  const int64_t G0 = total * blockIdx.x / gridDim.x, G1 = total * (blockIdx.x + 1) / gridDim.x;
  if (G0 >= G1) return;
  const int64_t img0 = G0 / ntile;
  const int nimg = int((G1 - 1) / ntile - img0 + 1);

  if (warp == 0) {
    // TMEM: T slots of SLOT_COLS columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(lay.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid < 2 * T) tc::mbar_init(&mbar[tid], 1);  // slot s: mbar[s] (first N chain), mbar[T + s]
  if (shared_tab) build_coord_tables(a, aug, 0, tabs, tabs + ((a.out_w + 3) & ~3), tid, NT);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // 16-byte vector stores of full warps: f32 NCHW / NHWC need hw % 4 == 0,
  // bf16 NCHW hw % 8 == 0 (u8 and the rest store per value)
  const bool vec_store = (a.dtype == RINR_OUT_F32 && a.hw % 4 == 0) ||
                         (a.dtype == RINR_OUT_BF16 && a.layout == RINR_LAYOUT_NCHW && a.hw % 8 == 0);
  uint32_t mma_phase = 0;  // parity of this epilogue warp's slot mbarrier

  for (int c0 = 0; c0 < nimg; c0 += lay.maxi) {
    const int ni = min(lay.maxi, nimg - c0);
    const int64_t cimg = img0 + c0;
    // =============================== phase 1 =================================
    for (int i = warp; i < ni; i += NW) {
      const int64_t id = ids[cimg + i];
      const bool ok = id >= 0 && id < sv.n;
      if (lane == 0) {
        if (!ok) flag_bad_id(status, n, cimg + i);
        metaid[i] = ok ? id : -1;
      }
      if (!ok) continue;
      uint64_t off;
      uint32_t bytes;
      slot_of(sv, id, off, bytes);
      const uint8_t* src = sv.blob + off;
      uint8_t* dst = recs + size_t(i) * lay.rec_bytes;
      // (32 lanes x 16-B cp.async: one TMA bulk copy per 13.6-KB record measured
      // 1.7% slower here, 133.8 vs 136.0 K img/s on c3; decode_persist uses it)
      for (uint32_t k = lane; k < bytes / 16; k += 32) cp_async16(dst + 16 * k, src + 16 * k);
    }
    cp_async_commit();
    for (int i = tid; i < ni * lay.net_bytes / 16; i += NT) reinterpret_cast<uint4*>(nets)[i] = make_uint4(0, 0, 0, 0);
    if (!shared_tab)
      for (int i = 0; i < ni; ++i) {
        float* tab = tabs + i * lay.tab_floats;
        build_coord_tables(a, aug, cimg + i, tab, tab + ((a.out_w + 3) & ~3), tid, NT);
      }
    cp_async_wait_all();
    __syncthreads();
    for (int q = warp; q < ni * NL; q += NW) {
      const int i = q / NL, l = q - i * NL;
      if (metaid[i] < 0) continue;
      const uint32_t* lo = reinterpret_cast<const uint32_t*>(recs + size_t(i) * lay.rec_bytes);
      const uint8_t* rec = recs + size_t(i) * lay.rec_bytes + sv.hdr_bytes;
      const int fi = l == 0 ? 2 : HID, fo = l == NL - 1 ? 3 : HID;
      const DLayer L = parse_layer(rec, lo[l], lo[l + 1], fi, fo);
      if (L.form != FORM_DENSE) {
        uint32_t* words = pfx + i * lay.pfx_words + l * 2 * KW;
        build_bit_prefix(rec, L, words, words + KW, lane);
      }
    }
    __syncthreads();
    {
      constexpr int P0 = 3 * HID, PH = HID * HID + HID, PO = 3 * HID + 3;
      constexpr int PALL = P0 + (NL - 2) * PH + PO;
      for (int q = tid; q < ni * PALL; q += NT) {
        const int i = q / PALL;
        int e = q - i * PALL;
        if (metaid[i] < 0) continue;
        int l, o, k;
        bool is_bias;
        if (e < P0) {
          l = 0;
          is_bias = e >= 2 * HID;
          o = is_bias ? e - 2 * HID : e / 2;
          k = is_bias ? 0 : e - 2 * o;
        } else if (e < P0 + (NL - 2) * PH) {
          e -= P0;
          const int h = e / PH;
          e -= h * PH;
          l = 1 + h;
          is_bias = e >= HID * HID;
          o = is_bias ? e - HID * HID : e / HID;
          k = is_bias ? 0 : e - HID * o;
        } else {
          e -= P0 + (NL - 2) * PH;
          l = NL - 1;
          is_bias = e >= 3 * HID;
          o = is_bias ? e - 3 * HID : e / HID;
          k = is_bias ? 0 : e - HID * o;
        }
        const uint32_t* lo = reinterpret_cast<const uint32_t*>(recs + size_t(i) * lay.rec_bytes);
        const uint8_t* rec = recs + size_t(i) * lay.rec_bytes + sv.hdr_bytes;
        const int fi = l == 0 ? 2 : HID, fo = l == NL - 1 ? 3 : HID;
        const DLayer L = parse_layer(rec, lo[l], lo[l + 1], fi, fo);
        const uint32_t* words = pfx + i * lay.pfx_words + l * 2 * KW;
        const bool hidden = l > 0 && l < NL - 1;
        const bool int_b = hidden && int_b_exact(L);
        Net net(nets + size_t(i) * lay.net_bytes);
        if (is_bias) {
          const float bb = dq_bias(rec, L, o);
          if (l == 0) net.l0[o * 4 + 2] = __fmul_rn(omega, bb);
          else if (hidden) net.biasH[(l - 1) * C::KP + o] = __fmul_rn(omega, bb);
          else net.biasO[o] = bb;
          if (hidden && o == 0) {
            net.modeH[l - 1] = int_b ? 1 : 0;
            net.scaleH[l - 1] = int_b ? __double2float_rn(double(omega) * L.scale) : 1.0f;
          }
        } else {
          const int j = o * fi + k;
          if (l == 0) {
            net.l0[o * 4 + k] = __fmul_rn(omega, dq_weight(rec, L, words, words + KW, j));
          } else if (hidden) {
            uint8_t* bh = net.bh_hi + (l - 1) * C::BH_BYTES;
            uint8_t* bl = net.bh_lo + (l - 1) * C::BH_BYTES;
            if (int_b) Net::put(bh, INTB ? nullptr : bl, o, k, dq_int(rec, L, words, words + KW, j), 0.0f);
            else if (!INTB) Net::put_split(bh, bl, o, k, __fmul_rn(omega, dq_weight(rec, L, words, words + KW, j)));
          } else {
            Net::put_split(net.bo_hi, net.bo_lo, o, k, dq_weight(rec, L, words, words + KW, j));
          }
        }
      }
    }
    tc::fence_async_smem();  // B matrices are read by the tensor core (async proxy)
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (c0 == 0) {
      if (overlap) pdl_wait();
      pdl_trigger();
    }

    // =============================== phase 2 =================================
    const int64_t cbase = cimg * ntile;
    const int ts = int((G0 > cbase ? G0 : cbase) - cbase);
    const int te = int((G1 < cbase + int64_t(ni) * ntile ? G1 : cbase + int64_t(ni) * ntile) - cbase);
    const int nt_chunk = te - ts;
    const int rounds = (nt_chunk + T - 1) / T;

    {
      // ------------------------------ epilogue warps --------------------------
      const int s = warp >> 2;          // tile slot
      const int q = warp & 3;           // TMEM lane quarter
      const int row = q * 32 + lane;    // pixel row within the tile
      constexpr int SLOT = C::slot_cols(X3);
      const uint32_t tacc = tmem_base + uint32_t(s * SLOT) + (uint32_t(q * 32) << 16);
      const uint32_t tahi = tacc + C::ahi_col(X3), talo = tacc + C::alo_col();
      const bool issuer = q == 0 && lane == 0;
      const uint32_t dslot = tmem_base + uint32_t(s * SLOT);
      RINR_DCHECK((s + 1) * SLOT <= lay.tmem_cols);
      const float invW = 1.0f / float(a.out_w);
      for (int r = 0; r < rounds; ++r) {
        const int t = ts + r * T + s;
        if (t >= te) break;
        const int i = t / ntile;
        const int64_t img = cimg + i;
        const Net net(nets + size_t(i) * lay.net_bytes);
        const float* colx = shared_tab ? tabs : tabs + i * lay.tab_floats;
        const float* rowy = colx + ((a.out_w + 3) & ~3);
        const int p = (t - i * ntile) * 128 + row;
        const bool inside = p < a.hw;
        int pr = int(float(p) * invW);
        int pc = p - pr * a.out_w;
        if (pc >= a.out_w) { pc -= a.out_w; ++pr; }
        if (pc < 0) { pc += a.out_w; --pr; }
        const float x = colx[inside ? pc : 0], y = rowy[inside ? pr : 0];
        RINR_TC_STAMP(s, r, 0, 0);  // tile start
        // ---- layer 0 on FFMA -> A row (TMEM) ----
#pragma unroll
        for (int ks = 0; ks < C::KS; ++ks) {
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {  // two columns per FFMA2 pair
              const int col = ks * 16 + half * 8 + e;
              const float4 w = reinterpret_cast<const float4*>(net.l0)[col];
              const float4 w2 = reinterpret_cast<const float4*>(net.l0)[col + 1];
              const float2 z = ffma2(make_float2(w.y, w2.y), make_float2(y, y),
                                     ffma2(make_float2(w.x, w2.x), make_float2(x, x), make_float2(w.z, w2.z)));
              v[e] = col < HID ? __sinf(z.x) : 0.0f;
              v[e + 1] = col + 1 < HID ? __sinf(z.y) : 0.0f;
            }
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) pack_act<X3>(v[2 * i2], v[2 * i2 + 1], hi[half * 4 + i2], lo[half * 4 + i2]);
          }
          tc::tmem_st8(tahi + uint32_t(ks * 8), hi);
          if (X3) tc::tmem_st8(talo + uint32_t(ks * 8), lo);
        }
        tc::tmem_wait_st();
        tc::fence_before();
        tc::bar_sync(1 + s, 4 * 32);  // the slot's A operand is complete
        tc::fence_after();
        RINR_TC_STAMP(s, r, 0, 2);
        if (kWarpIssue ? q == 0 : issuer) issue_layer<HID, NL, X3, INTB>(net, dslot, 0, &mbar[s], &mbar[T + s]);
        RINR_TC_STAMP(s, r, 0, 3);
        // ---- hidden layers: TMEM -> sine -> A row ----
        // several layers per trip: the compiler overlaps one layer's tail with
        // the next layer's wait / load.  Measured on c3 (8 hidden layers):
        // fp32 1 / 2 / 4 / 8 per trip = 149.4 / 153.2 / 154.2 / 148.9 K img/s,
        // bf16 180.8 / 185.5 / 186.7 / 190.0 K img/s
        constexpr int LUNROLL = X3 ? 4 : 8;
#pragma unroll LUNROLL
        for (int l = 0; l < NL - 2; ++l) {
          RINR_TC_STAMP(s, r, l + 1, 0);
          tc::mbar_wait(&mbar[s], mma_phase);
          RINR_TC_STAMP(s, r, l + 1, 1);
          tc::fence_after();
          const float sc = net.scaleH[l];
          const float* bias = net.biasH + l * C::KP;
          constexpr int CV = (HID + 7) / 8;  // chunks holding real columns
          float v[CV][8];
          using SN = SplitN<HID, NL, INTB>;
          // SN::ON: chunks of the first N chain, waited for on mbar[s]; the
          // rest on mbar[T + s] once the first K steps' sines are done.
          // Otherwise the first K step's columns are loaded and waited for
          // alone while the rest stay in flight.
          constexpr int CA = SN::ON ? (SN::NA / 8 < CV ? SN::NA / 8 : CV) : (CV < 2 ? CV : 2);
          constexpr int KSA = SN::ON ? SN::NA / 16 : 1;  // K steps served by the first chunks
#pragma unroll
          for (int cc = 0; cc < CA; ++cc) tc::tmem_ld8(tacc + uint32_t(cc * 8), v[cc]);
          tc::tmem_wait_ld();
#pragma unroll
          for (int cc = 0; cc < CA; ++cc) tc::pin8(v[cc]);
          if constexpr (!SN::ON) {
#pragma unroll
            for (int cc = CA; cc < CV; ++cc) tc::tmem_ld8(tacc + uint32_t(cc * 8), v[cc]);
          }
#pragma unroll
          for (int ks = 0; ks < C::KS; ++ks) {
            if (ks == KSA && CA < CV) {
              if constexpr (SN::ON) {
                tc::mbar_wait(&mbar[T + s], mma_phase);
                tc::fence_after();
#pragma unroll
                for (int cc = CA; cc < CV; ++cc) tc::tmem_ld8(tacc + uint32_t(cc * 8), v[cc]);
              }
              tc::tmem_wait_ld();
#pragma unroll
              for (int cc = CA; cc < CV; ++cc) tc::pin8(v[cc]);
            }
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              const int cchunk = 2 * ks + half;
              float u[8];
              if (cchunk < CV) {
                const float4 b0 = reinterpret_cast<const float4*>(bias)[2 * cchunk];
                const float4 b1 = reinterpret_cast<const float4*>(bias)[2 * cchunk + 1];
                const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int e = 0; e < 8; e += 2) {  // packed scale + bias (FFMA2)
                  const float* vc = v[cchunk < CV ? cchunk : 0];
                  const float2 z = ffma2(make_float2(vc[e], vc[e + 1]), make_float2(sc, sc), make_float2(bb[e], bb[e + 1]));
                  u[e] = cchunk * 8 + e < HID ? __sinf(z.x) : 0.0f;
                  u[e + 1] = cchunk * 8 + e + 1 < HID ? __sinf(z.y) : 0.0f;
                }
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) u[e] = 0.0f;
              }
#pragma unroll
              for (int i2 = 0; i2 < 4; ++i2) pack_act<X3>(u[2 * i2], u[2 * i2 + 1], hi[half * 4 + i2], lo[half * 4 + i2]);
            }
            tc::tmem_st8(tahi + uint32_t(ks * 8), hi);
            if (X3) tc::tmem_st8(talo + uint32_t(ks * 8), lo);
          }
          if constexpr (SN::ON) {
            if (CA >= CV) tc::mbar_wait(&mbar[T + s], mma_phase);  // keep both barriers' phases in step
          }
          // the parity flips here, at the end of the epilogue, not right after
          // the wait: measured +7% (fp32) / +2.4% (bf16) from the schedule
          mma_phase ^= 1u;
          tc::tmem_wait_st();
          tc::fence_before();
          tc::bar_sync(1 + s, 4 * 32);
          tc::fence_after();
          RINR_TC_STAMP(s, r, l + 1, 2);
          if (kWarpIssue ? q == 0 : issuer) issue_layer<HID, NL, X3, INTB>(net, dslot, l + 1, &mbar[s], &mbar[T + s]);
          RINR_TC_STAMP(s, r, l + 1, 3);
        }
        // ---- output layer ----
        RINR_TC_STAMP(s, r, NL - 1, 0);
        tc::mbar_wait(&mbar[s], mma_phase);
        if constexpr (SplitN<HID, NL, INTB>::ON) tc::mbar_wait(&mbar[T + s], mma_phase);
        RINR_TC_STAMP(s, r, NL - 1, 1);
        mma_phase ^= 1u;
        tc::fence_after();
        float o[8];
        tc::tmem_ld8(tacc, o);
        tc::tmem_wait_ld();
        tc::fence_before();  // TMEM reads done before the next tile's MMA overwrites it
        // epilogue: clamp (decoder.py:35), normalise, then the warp's 32
        // consecutive pixels x 3 channels go through a shared-memory stage
        // (the free phase-1 scratch) and out as 16-byte vector stores
        float* sw = reinterpret_cast<float*>(smem) + warp * 96;  // [ch][32 px]
        RINR_DCHECK(in_smem(sw, 96 * 4) && warp * 96 * 4 + 384 <= lay.region0);
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          float vv = __saturatef(o[ch] + net.biasO[ch]);
          if (!a.identity) {
            const float m = ch == 0 ? a.mean[0] : (ch == 1 ? a.mean[1] : a.mean[2]);
            const float sd = ch == 0 ? a.stdv[0] : (ch == 1 ? a.stdv[1] : a.stdv[2]);
            vv = __fdiv_rn(__fsub_rn(vv, m), sd);
          }
          sw[ch * 32 + lane] = vv;
        }
        __syncwarp();
        const int p0 = p - lane;  // first pixel of the warp (a multiple of 32)
        if (vec_store && p0 + 32 <= a.hw) {
          if (a.layout == RINR_LAYOUT_NCHW && a.dtype == RINR_OUT_BF16) {
            if (lane < 12) {  // channel lane/4, 8 pixels each
              const int ch = lane >> 2, part = lane & 3;
              const float4 u = *reinterpret_cast<const float4*>(sw + ch * 32 + part * 8);
              const float4 v = *reinterpret_cast<const float4*>(sw + ch * 32 + part * 8 + 4);
              uint4 pk;
              pk.x = bf2_bits(__floats2bfloat162_rn(u.x, u.y));
              pk.y = bf2_bits(__floats2bfloat162_rn(u.z, u.w));
              pk.z = bf2_bits(__floats2bfloat162_rn(v.x, v.y));
              pk.w = bf2_bits(__floats2bfloat162_rn(v.z, v.w));
              RINR_DCHECK((img * 3 + ch) * int64_t(a.hw) + p0 + part * 8 + 8 <= a.out_elems);
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + (img * 3 + ch) * int64_t(a.hw) + p0 +
                                        part * 8) = pk;
            }
          } else if (a.layout == RINR_LAYOUT_NCHW) {  // f32
            if (lane < 24) {
              const int ch = lane >> 3, part = lane & 7;
              RINR_DCHECK((img * 3 + ch) * int64_t(a.hw) + p0 + part * 4 + 4 <= a.out_elems);
              *reinterpret_cast<float4*>(static_cast<float*>(out) + (img * 3 + ch) * int64_t(a.hw) + p0 + part * 4) =
                  *reinterpret_cast<const float4*>(sw + ch * 32 + part * 4);
            }
          } else {  // NHWC f32: 96 interleaved values
            if (lane < 24) {
              float v4[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int e = 4 * lane + k, px = e / 3, ch = e - 3 * px;
                v4[k] = sw[ch * 32 + px];
              }
              RINR_DCHECK((img * a.hw + p0) * 3 + 4 * lane + 4 <= a.out_elems);
              *reinterpret_cast<float4*>(static_cast<float*>(out) + (img * a.hw + p0) * 3 + 4 * lane) =
                  make_float4(v4[0], v4[1], v4[2], v4[3]);
            }
          }
        } else if (inside) {
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) store_value(a, out, img, p, ch, sw[ch * 32 + lane]);
        }
        __syncwarp();
        RINR_TC_STAMP(s, r, NL, 0);  // tile stored
      }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
  }
  __syncthreads();
  if (warp == 0) {
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(lay.tmem_cols)
                 : "memory");
  }
}

}  // namespace rinr
