// Persistent two-phase batched decode (uniform-width SIREN).
//
// Grid = one CTA per SM.  The batch is cut into pixel groups (NB blocks of
// 16 pixels of one image); CTA c owns the contiguous group range
// [c*T/G, (c+1)*T/G), so every CTA gets the same work to within one group and
// visits at most ceil(n/G)+1 images.  Those images are processed in chunks of
// up to `maxi` images (what fits in shared memory), each in two phases:
//
//   phase 1 (all warps): fetch the chunk's record metadata, cp.async every
//     record's bytes from the HBM store into shared memory, build the kept-bit
//     prefix tables (one warp per sparse layer), then dequantise all entries of
//     all images in parallel — bit-exact with archive.materialize — straight
//     into the MMA operand layout (mma_chain.cuh NetView).
//   phase 2 (all warps): round-robin over the chunk's pixel groups; each warp
//     runs the register-resident mma.sync layer chain and stores through a
//     per-warp stage with 16-byte vector stores.
#pragma once

#include <type_traits>

#include "mma_chain.cuh"

namespace rinr {

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  RINR_DCHECK(in_smem(smem_dst, 16));
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// Record staging by the TMA bulk engine: one cp.async.bulk per record slot
// (UBLKCP in SASS), completion counted in bytes on a shared mbarrier.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bulk_mbar_init(uint64_t* mbar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(mbar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// expect `bytes` more and start the copy global -> shared (16-B aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  RINR_DCHECK(in_smem(dst, bytes) && (bytes & 15u) == 0);
  // the slot may have been read through the generic proxy (previous chunk)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(mbar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(mbar))
               : "memory");
}
// L2 prefetch of a record slot by the bulk engine (no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// the single arrival of the phase (after every expect_tx of the phase was issued)
__device__ __forceinline__ void bulk_mbar_arrive(uint64_t* mbar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(mbar))
               : "memory");
}
// Per-image network readiness (phase 1 -> phase 2): count = dequant tasks of
// the image; each task's lane 0 arrives (release) after the warp's fragment
// writes, phase-2 warps wait (acquire) before their first group of the image.
__device__ __forceinline__ void ready_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void ready_arrive(uint64_t* mbar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(mbar))
               : "memory");
}
__device__ __forceinline__ void bulk_mbar_wait(uint64_t* mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "BULK_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra BULK_WAIT_%=;\n\t}\n" ::"r"(smem_addr(mbar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// Programmatic dependent launch: wait for the preceding grid / let the next start.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifdef RINR_DEV_KNOBS
// Development timeline (RINR_DEV_KNOBS builds only, tools/dev_timeline.py):
// %globaltimer of each CTA's thread 0 at the phase boundaries of the last 4
// launches, and clock64 durations of each warp's first dequant task.
__device__ unsigned long long g_dev_t[4][512][8];
__device__ unsigned long long g_dev_task[512][16][2];
__device__ __forceinline__ void dev_stamp(int overlap, int stage) {
  if (threadIdx.x == 0 && blockIdx.x < 512) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dev_t[(overlap >> 4) & 3][blockIdx.x][stage] = t;
  }
}
#else
__device__ __forceinline__ void dev_stamp(int, int) {}
#endif

struct PersistLayout {
  int maxi;        // images per chunk
  int net_words;   // per image
  int tab_floats;  // per table set: round4(W) + round4(H + 1)
  int rec_bytes;   // per image record slot (16-B multiple)
  int pfx_words;   // per image: NL layers x (bit words + prefix)
};

// Per-image operands a warp keeps in registers while decoding that image.
template <int HID, int NL>
struct ImgRegs {
  using C = MmaCfg<HID, NL>;
  static constexpr int K1 = C::NH == 1 ? C::KT : 1;
  static constexpr int N1 = C::NH == 1 ? C::NT : 1;
  // Narrow nets keep the layer-0 and output operands in registers; wide nets
  // (KT > 1) read them from shared memory per group to free ~60 registers.
  static constexpr bool REG_IO = C::KT == 1;
  static constexpr int KR = REG_IO ? C::KT : 1;
  float4 w0[KR][4];
  uint4 bo[KR];
  float bias_o;  // output tq's bias (output c sits in C-fragment column 2c)
  uint4 bh1[K1][N1];  // hidden layer 1 fragments (only when it is the only hidden layer)
  float2 bb1[N1];
  float sc1;
  bool int1;
  float mean0, std0;  // epilogue constants of this lane's channel tq (tq < 3)
  bool ident;

  __device__ __forceinline__ void set_norm(const DecodeArgs& a, int lane) {
    const int tq = lane & 3;
    ident = a.identity != 0;
    // static indices: a dynamically indexed parameter array would be copied to the stack
    mean0 = tq == 1 ? a.mean[1] : (tq == 2 ? a.mean[2] : a.mean[0]);
    std0 = tq == 1 ? a.stdv[1] : (tq == 2 ? a.stdv[2] : a.stdv[0]);
  }

  __device__ __forceinline__ void load(const NetView<HID, NL>& net, int lane) {
    const int tq = lane & 3;
    if constexpr (REG_IO) {
#pragma unroll
      for (int t = 0; t < C::KT; ++t)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          w0[t][q] = reinterpret_cast<const float4*>(net.l0)[16 * t + 2 * tq + (q & 1) + 8 * (q >> 1)];
#pragma unroll
      for (int t = 0; t < C::KT; ++t) bo[t] = reinterpret_cast<const uint4*>(net.fragO)[t * 32 + lane];
    }
    bias_o = net.biasO[tq];  // biasO[3] is zero
    if constexpr (C::NH == 1) {
#pragma unroll
      for (int t = 0; t < C::KT; ++t)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) bh1[t][j] = reinterpret_cast<const uint4*>(net.fragH)[(t * C::NT + j) * 32 + lane];
#pragma unroll
      for (int j = 0; j < C::NT; ++j) bb1[j] = *reinterpret_cast<const float2*>(net.biasH + 8 * j + 2 * tq);
      int1 = net.modeH[0] != 0;
      sc1 = net.scaleH[0];
    }
  }
};

// One fragment-owner dequant task of one record (slot = the record's shared
// copy: layer-offset header, then the body at sv.hdr_bytes): h = 0 writes
// layer 0 + the output layer, h = 1..NL-2 hidden layer h, straight into the
// MMA operand layout of `net` (shared or global memory).  Every lane writes
// exactly the fragment words it owns, padding included (no zero fill), with
// values bit-exact to archive.materialize (archive.py:278-325).
template <int HID, int NL, bool INTB>
__device__ __forceinline__ void frag_task(const StoreView& sv, const uint8_t* slot, int h, NetView<HID, NL> net,
                                          float omega, int lane) {
  using C = MmaCfg<HID, NL>;
  const uint32_t* lo = reinterpret_cast<const uint32_t*>(slot);
  const uint8_t* rec = slot + sv.hdr_bytes;
  if (h == 0) {
    const DLayer L0 = parse_layer(rec, lo[0], lo[1], 2, HID);
    const DLayer LO = parse_layer(rec, lo[NL - 1], lo[NL], HID, 3);
    const WarpBits B0 = warp_bits(rec, L0, lane), BO = warp_bits(rec, LO, lane);
    const ValueRecipe R0 = value_recipe(L0), RO = value_recipe(LO);
    // layer 0: lane c -> {omega w[c][0], omega w[c][1], omega b[c], 0}
    auto layer0 = [&](auto kind) {
      constexpr int K = decltype(kind)::value;
      const int c = lane < C::KP ? lane : 0;
      const float w0 = value_at<false, K>(rec, R0, B0, c < HID ? 2 * c : 0);
      const float w1 = value_at<false, K>(rec, R0, B0, c < HID ? 2 * c + 1 : 0);
      if (lane < C::KP) {
        float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < HID) {
          e.x = __fmul_rn(omega, w0);
          e.y = __fmul_rn(omega, w1);
          e.z = __fmul_rn(omega, dq_bias(rec, L0, c));
        }
        reinterpret_cast<float4*>(net.l0)[c] = e;
      }
    };
    const int k0 = value_kind(L0);
    if (k0 == VK_F32) layer0(std::integral_constant<int, VK_F32>{});
    else layer0(std::integral_constant<int, VK_GEN>{});
    auto outl = [&](auto kind) {
      constexpr int K = decltype(kind)::value;
#pragma unroll
      for (int t = 0; t < C::KT; ++t)
        reinterpret_cast<uint4*>(net.fragO)[t * 32 + lane] =
            frag_words<false, K, true>(rec, RO, BO, HID, 3, t, 0, 1.0f, lane);
    };
    const int ko = value_kind(LO);
    if (ko == VK_F32) outl(std::integral_constant<int, VK_F32>{});
    else outl(std::integral_constant<int, VK_GEN>{});
    if (lane < 8) net.biasO[lane] = lane < 3 ? dq_bias(rec, LO, lane) : 0.0f;
  } else {
    const int l = h;
    const DLayer L = parse_layer(rec, lo[l], lo[l + 1], HID, HID);
    const WarpBits B = warp_bits(rec, L, lane);
    const ValueRecipe R = value_recipe(L);
    const bool int_b = INTB || int_b_exact(L);
    uint4* fr = reinterpret_cast<uint4*>(net.fragH + (l - 1) * C::KT * C::NT * 32 * 4);
    if (int_b) {
#pragma unroll
      for (int t = 0; t < C::KT; ++t)
#pragma unroll
        for (int j = 0; j < C::NT; ++j)
          fr[(t * C::NT + j) * 32 + lane] = frag_words<true>(rec, R, B, HID, HID, t, j, omega, lane);
    } else {
      auto hid = [&](auto kind) {
        constexpr int K = decltype(kind)::value;
#pragma unroll
        for (int t = 0; t < C::KT; ++t)
#pragma unroll
          for (int j = 0; j < C::NT; ++j)
            fr[(t * C::NT + j) * 32 + lane] = frag_words<false, K>(rec, R, B, HID, HID, t, j, omega, lane);
      };
      if (value_kind(L) == VK_F32) hid(std::integral_constant<int, VK_F32>{});
      else hid(std::integral_constant<int, VK_GEN>{});
    }
    static_assert(C::NT * 8 <= 32, "one bias entry per lane");
    if (lane < C::NT * 8)
      net.biasH[(l - 1) * C::NT * 8 + lane] = lane < HID ? __fmul_rn(omega, dq_bias(rec, L, lane)) : 0.0f;
    if (lane == 0) {
      net.modeH[l - 1] = int_b ? 1 : 0;
      net.scaleH[l - 1] = int_b ? __double2float_rn(double(omega) * L.scale) : 1.0f;
    }
  }
}

// Phase-2 specialisation, chosen once per launch (warp-uniform):
//   ALIGNED : out_w is a multiple of the group width, so a group lies inside one
//             image row and every group is full
//   STORE   : 1 NCHW f32, 2 NCHW bf16, 3 NHWC f32 (16-byte vector stores,
//             ALIGNED only), 0 any dtype/layout (scalar stores)
// Each mode is its own kernel instantiation (one large inlined loop per
// kernel keeps ptxas from spilling).
//   INTB    : every hidden layer of every record in the store is affine8
//             (integer-code B operand; compile-time, no branch around mma.sync)
//   SEP     : separable layer 0 (out_w == group width, narrow net, MUFU sine):
//             sin(a x + r(y)) = sin(a x) cos(r) + cos(a x) sin(r), with the
//             per-image column terms held in registers and the per-row terms
//             computed once per row by the warp (one sine per lane)
template <bool ALIGNED_, int STORE_, bool INTB_ = false, bool SEP_ = false>
struct Mode {
  static constexpr bool ALIGNED = ALIGNED_;
  static constexpr int STORE = STORE_;
  static constexpr bool INTB = INTB_;
  static constexpr bool SEP = SEP_;
};

// Column terms of the separable layer 0 for one image (SEP mode): the lane's
// four pixel columns c = 16 bk + 8 h + g and four units u(q) = 2 tq + (q & 1)
// + 8 (q >> 1): sa = sin(omega w0[u] x_c), ca = cos(omega w0[u] x_c); plus
// this lane's row-term unit (lane & 15): omega w1, omega b (+ pi/2 on the
// cosine lanes 16..31).
struct SepRegs {
  float sa[2][2][4], ca[2][2][4];
  float w1, b1;
  int slot;  // this lane's row-term slot (sep_row_slot)
};

// Row terms of one output row y for the separable layer 0: lane (u = lane & 15,
// f = lane >> 4) evaluates sin(r_u + f pi/2), r_u = omega (w1[u] y + b[u]), and
// stores it at [pair u/2][f][u&1] so that one 16-byte load returns
// {sin r_2p, sin r_2p+1, cos r_2p, cos r_2p+1}.
// (The cosine lanes carry pi/2 in S.b1.)
__device__ __forceinline__ int sep_row_slot(int lane) {
  const int u = lane & 15, f = lane >> 4;
  return 4 * (u >> 1) + 2 * f + (u & 1);
}
__device__ __forceinline__ void sep_row_terms(const SepRegs& S, float y, float* rowt, int slot) {
  rowt[slot] = __sinf(fmaf(S.w1, y, S.b1));
}

// NCHW f32 output (STORE 1) is stored straight from the output MMA's C
// fragment: output c sits in column 2c, so lane (g, tq < 3) holds channel tq
// at pixels g, g + 8 of each 16-pixel block and writes them with 4 STG per
// group; each instruction covers whole 32-byte sectors (8 lanes x 4 B per
// channel).  No stage round trip (was 8 STS + LDS.128 + STG.128).
#ifdef RINR_STAGED_STORE1
constexpr bool DIRECT_STORE1 = false;
#else
constexpr bool DIRECT_STORE1 = true;
#endif

// Per-lane store addressing, fixed for a launch.
struct StoreLane {
  int soff[4];   // stage indices this lane reads
  int64_t goff;  // element offset of this lane's vector within an image group
  bool active;
};

template <int NB, int STORE>
__device__ __forceinline__ StoreLane make_store_lane(const DecodeArgs& a, int lane) {
  constexpr int GPX = NB * 16;
  StoreLane L{};
  if constexpr (STORE == 1 && DIRECT_STORE1) {  // NCHW f32 straight from the C fragment
    const int g = lane >> 2, tq = lane & 3;
    L.active = tq < 3;  // channel tq
    L.goff = int64_t(tq) * a.hw + g;
  } else if constexpr (STORE == 1) {  // NCHW f32: lane -> (channel, float4 of the group)
    constexpr int V = GPX / 4;
    const int ch = lane / V, part = lane - ch * V;
    L.active = lane < 3 * V;
    L.soff[0] = ch * GPX + part * 4;
    L.goff = int64_t(ch) * a.hw + part * 4;
  } else if constexpr (STORE == 2) {  // NCHW bf16: lane -> (channel, 8 values)
    constexpr int V = GPX / 8;
    const int ch = lane / V, part = lane - ch * V;
    L.active = lane < 3 * V;
    L.soff[0] = ch * GPX + part * 8;
    L.goff = int64_t(ch) * a.hw + part * 8;
  } else if constexpr (STORE == 3) {  // NHWC f32: lane -> 4 consecutive interleaved values
    constexpr int V = 3 * GPX / 4;
    L.active = lane < V;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = 4 * lane + q, px = e / 3, ch = e - 3 * px;
      L.soff[q] = ch * GPX + px;
    }
    L.goff = 4 * lane;
  }
  return L;
}

// One group: NB blocks of 16 pixels of image `img`, pixels [pbase, pbase+16*NB).
// `obase` is the element offset of image img in the output.
template <int HID, int NL, bool X3, bool ACCURATE, int NB, class M>
__device__ __forceinline__ void decode_group(const NetView<HID, NL>& net, const ImgRegs<HID, NL>& R,
                                             const float* colx, const float* rowy, const DecodeArgs& a,
                                             void* __restrict__ out, int64_t img, int64_t obase, int pbase,
                                             int rb, int cb, float* stage, const StoreLane& SL, int lane,
                                             const SepRegs& S, const float* rowt, float* rowt_next, bool next_row,
                                             int64_t gofs) {
  // gofs: element offset of this lane's vector store for the group (STORE 1-3)
  // (rb, cb): row / column of the group's first pixel
  using C = MmaCfg<HID, NL>;
  constexpr int GPX = NB * 16;
  constexpr bool ALIGNED = M::ALIGNED;
  const int g = lane >> 2, tq = lane & 3;
  const int W = a.out_w;

  uint32_t ah[NB][C::KT][4], al[NB][C::KT][4];
  if constexpr (M::SEP) {
    static_assert(C::KT == 1 && NB == 2, "separable layer 0: one k-tile, one 32-pixel row per group");
    // row terms of this group's row (written one group ahead), then per
    // pixel and unit s = sa * cos r + ca * sin r  (FMUL2 + FFMA2 per unit pair)
    const float4 r0 = reinterpret_cast<const float4*>(rowt)[tq];      // units 2tq, 2tq+1
    const float4 r1 = reinterpret_cast<const float4*>(rowt)[tq + 4];  // units 2tq+8, 2tq+9
    // next row's terms overlap this group (visible after the closing __syncwarp)
    if (next_row) sep_row_terms(S, rowy[rb + 1], rowt_next, S.slot);  // rowy[out_h] exists
#pragma unroll
    for (int bk = 0; bk < NB; ++bk) {
      float v[2][4];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float2 lo = ffma2(make_float2(S.sa[bk][h][0], S.sa[bk][h][1]), make_float2(r0.z, r0.w),
                                fmul2(make_float2(S.ca[bk][h][0], S.ca[bk][h][1]), make_float2(r0.x, r0.y)));
        const float2 hi = ffma2(make_float2(S.sa[bk][h][2], S.sa[bk][h][3]), make_float2(r1.z, r1.w),
                                fmul2(make_float2(S.ca[bk][h][2], S.ca[bk][h][3]), make_float2(r1.x, r1.y)));
        v[h][0] = lo.x;
        v[h][1] = lo.y;
        v[h][2] = hi.x;
        v[h][3] = hi.y;
      }
      pack_act<X3>(v[0][0], v[0][1], ah[bk][0][0], al[bk][0][0]);
      pack_act<X3>(v[1][0], v[1][1], ah[bk][0][1], al[bk][0][1]);
      pack_act<X3>(v[0][2], v[0][3], ah[bk][0][2], al[bk][0][2]);
      pack_act<X3>(v[1][2], v[1][3], ah[bk][0][3], al[bk][0][3]);
    }
  } else {
#pragma unroll
    for (int bk = 0; bk < NB; ++bk) {
      float xr[2], yr[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if constexpr (ALIGNED) {  // W a multiple of the group: the group lies inside one row
          xr[h] = colx[cb + 16 * bk + 8 * h + g];
          yr[h] = rowy[rb];
        } else {
          int c = cb + 16 * bk + 8 * h + g, r = rb;
          while (c >= W) { c -= W; ++r; }
          const bool inside = pbase + 16 * bk + 8 * h + g < a.hw;
          xr[h] = colx[inside ? c : 0];
          yr[h] = rowy[inside ? r : 0];
        }
      }
#pragma unroll
      for (int t = 0; t < C::KT; ++t) {
        float s[2][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool pad = 16 * t + 8 * (q >> 1) >= HID;  // whole slot is padding (compile time)
          float4 w;
          if constexpr (ImgRegs<HID, NL>::REG_IO) w = R.w0[t][q];
          else w = reinterpret_cast<const float4*>(net.l0)[16 * t + 2 * tq + (q & 1) + 8 * (q >> 1)];
          if constexpr (ALIGNED) {
            // the whole group is one image row: omega*(w1*y + b) once per unit
            const float yb = fmaf(w.y, yr[0], w.z);
            const float2 z = ffma2(make_float2(xr[0], xr[1]), make_float2(w.x, w.x), make_float2(yb, yb));
            s[0][q] = pad ? 0.0f : sine<ACCURATE>(z.x);
            s[1][q] = pad ? 0.0f : sine<ACCURATE>(z.y);
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) s[h][q] = pad ? 0.0f : sine<ACCURATE>(fmaf(w.y, yr[h], fmaf(w.x, xr[h], w.z)));
          }
        }
        pack_act<X3>(s[0][0], s[0][1], ah[bk][t][0], al[bk][t][0]);
        pack_act<X3>(s[1][0], s[1][1], ah[bk][t][1], al[bk][t][1]);
        pack_act<X3>(s[0][2], s[0][3], ah[bk][t][2], al[bk][t][2]);
        pack_act<X3>(s[1][2], s[1][3], ah[bk][t][3], al[bk][t][3]);
      }
    }
  }
  // ---- hidden layers ---------------------------------------------------------
#pragma unroll 1
  for (int hl = 0; hl < C::NH; ++hl) {
    const uint32_t* fr = net.fragH + hl * C::KT * C::NT * 32 * 4;
    const bool int_b = M::INTB || (C::NH == 1 ? R.int1 : net.modeH[hl] != 0);
    const float sc = C::NH == 1 ? R.sc1 : net.scaleH[hl];
    float acc[NB][C::NT][4];  // first k-tile's MMA starts from zero (RZ accumulator)
    // int_b is warp-uniform: two straight-line MMA sequences instead of a
    // predicated mma.sync (which would still issue and force warp syncs)
    auto mma_layer = [&](auto with_lo) {
#pragma unroll
      for (int t = 0; t < C::KT; ++t) {
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          uint4 bf;
          if constexpr (C::NH == 1) bf = R.bh1[t][j];
          else bf = reinterpret_cast<const uint4*>(fr)[(t * C::NT + j) * 32 + lane];
#pragma unroll
          for (int bk = 0; bk < NB; ++bk) {
            if (t == 0) mma16816_z(acc[bk][j], ah[bk][t], bf.x, bf.y);
            else mma16816(acc[bk][j], ah[bk][t], bf.x, bf.y);
            if constexpr (X3) mma16816(acc[bk][j], al[bk][t], bf.x, bf.y);
            if constexpr (decltype(with_lo)::value) mma16816(acc[bk][j], ah[bk][t], bf.z, bf.w);
          }
        }
      }
    };
    if constexpr (M::INTB) {
      mma_layer(std::false_type{});
    } else {
      if (int_b) mma_layer(std::false_type{});
      else mma_layer(std::true_type{});
    }
    float2 bias[C::NT];
#pragma unroll
    for (int j = 0; j < C::NT; ++j) {
      if constexpr (C::NH == 1) bias[j] = R.bb1[j];
      else bias[j] = *reinterpret_cast<const float2*>(net.biasH + hl * C::NT * 8 + 8 * j + 2 * tq);
    }
#pragma unroll
    for (int bk = 0; bk < NB; ++bk) {
#pragma unroll
      for (int t = 0; t < C::KT; ++t) {
        float s[8];
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const int j = 2 * t + (e >> 2);
          if (j < C::NT) {
            const float2 z =
                ffma2(make_float2(acc[bk][j][e & 3], acc[bk][j][(e & 3) + 1]), make_float2(sc, sc), bias[j]);
            s[e] = sine<ACCURATE>(z.x);
            s[e + 1] = sine<ACCURATE>(z.y);
          } else {
            s[e] = s[e + 1] = 0.0f;
          }
        }
        pack_act<X3>(s[0], s[1], ah[bk][t][0], al[bk][t][0]);
        pack_act<X3>(s[2], s[3], ah[bk][t][1], al[bk][t][1]);
        pack_act<X3>(s[4], s[5], ah[bk][t][2], al[bk][t][2]);
        pack_act<X3>(s[6], s[7], ah[bk][t][3], al[bk][t][3]);
      }
    }
  }
  // ---- output layer + epilogue -------------------------------------------------
  float ov[NB][2];
#pragma unroll
  for (int bk = 0; bk < NB; ++bk) {
    // one accumulator, hi*Bhi + lo*Bhi + hi*Blo chained (no combine adds)
    float o[4];
#pragma unroll
    for (int t = 0; t < C::KT; ++t) {
      uint4 bo;
      if constexpr (ImgRegs<HID, NL>::REG_IO) bo = R.bo[t];
      else bo = reinterpret_cast<const uint4*>(net.fragO)[t * 32 + lane];
      if (t == 0) mma16816_z(o, ah[bk][t], bo.x, bo.y);
      else mma16816(o, ah[bk][t], bo.x, bo.y);
      if constexpr (X3) mma16816(o, al[bk][t], bo.x, bo.y);
      mma16816(o, ah[bk][t], bo.z, bo.w);
    }
    // o[0] = (px g, column 2tq = output tq), o[2] = (px g + 8, output tq); the
    // odd columns are zero padding.  Bias add + clamp (decoder.py:35) in one
    // saturating FADD.
    ov[bk][0] = __saturatef(o[0] + R.bias_o);
    ov[bk][1] = __saturatef(o[2] + R.bias_o);
  }
  if (!R.ident) {  // one uniform branch per group
#pragma unroll
    for (int bk = 0; bk < NB; ++bk)
#pragma unroll
      for (int e = 0; e < 2; ++e) ov[bk][e] = __fdiv_rn(__fsub_rn(ov[bk][e], R.mean0), R.std0);
  }
  if constexpr (M::STORE == 1 && DIRECT_STORE1) {
    if (SL.active) {
      float* p = static_cast<float*>(out) + gofs;  // channel tq, pixel pbase + g
      // logical element index of p[0] (the SEP loop passes a running pointer and gofs 0)
      RINR_DCHECK(img * 3 * int64_t(a.hw) + int64_t(tq) * a.hw + pbase + g >= 0 &&
                  img * 3 * int64_t(a.hw) + int64_t(tq) * a.hw + pbase + g + 16 * (NB - 1) + 8 < a.out_elems);
#pragma unroll
      for (int bk = 0; bk < NB; ++bk) {
        p[16 * bk] = ov[bk][0];
        p[16 * bk + 8] = ov[bk][1];
      }
    }
    __syncwarp();  // the SEP row terms written during this group become visible
    return;
  }
  if (tq < 3) {
#pragma unroll
    for (int bk = 0; bk < NB; ++bk)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        RINR_DCHECK(in_smem(stage + tq * GPX + 16 * bk + g + 8 * e, 4));
        stage[tq * GPX + 16 * bk + g + 8 * e] = ov[bk][e];
      }
  }
  __syncwarp();
  // ---- coalesced stores -------------------------------------------------------------
  if constexpr (M::STORE == 1) {
    if (SL.active) {
      RINR_DCHECK(gofs >= 0 && gofs + 4 <= a.out_elems);
      const float4 v = *reinterpret_cast<const float4*>(stage + SL.soff[0]);
      *reinterpret_cast<float4*>(static_cast<float*>(out) + gofs) = v;
    }
  } else if constexpr (M::STORE == 2) {
    if (SL.active) {
      RINR_DCHECK(gofs >= 0 && gofs + 8 <= a.out_elems);
      const float4 u = *reinterpret_cast<const float4*>(stage + SL.soff[0]);
      const float4 w = *reinterpret_cast<const float4*>(stage + SL.soff[0] + 4);
      uint4 pk;
      pk.x = bf2_bits(__floats2bfloat162_rn(u.x, u.y));
      pk.y = bf2_bits(__floats2bfloat162_rn(u.z, u.w));
      pk.z = bf2_bits(__floats2bfloat162_rn(w.x, w.y));
      pk.w = bf2_bits(__floats2bfloat162_rn(w.z, w.w));
      *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + gofs) = pk;
    }
  } else if constexpr (M::STORE == 3) {
    if (SL.active)
      RINR_DCHECK(gofs >= 0 && gofs + 4 <= a.out_elems);
    if (SL.active)
      *reinterpret_cast<float4*>(static_cast<float*>(out) + gofs) =
          make_float4(stage[SL.soff[0]], stage[SL.soff[1]], stage[SL.soff[2]], stage[SL.soff[3]]);
  } else {
    for (int i = lane; i < 3 * GPX; i += 32) {
      const int ch = i / GPX, q = i - ch * GPX;
      const int p = pbase + q;
      if (ALIGNED || p < a.hw) store_value(a, out, img, p, ch, stage[i]);
    }
  }
  __syncwarp();
}

// Phase 2 of one chunk: the warp's round-robin share of groups [gs, ge)
// (group indices relative to the chunk's first image cimg).
template <int HID, int NL, bool X3, bool ACCURATE, int NW, int NB, class M>
__device__ __forceinline__ void phase2_loop(const uint32_t* nets, const float* tabs, const PersistLayout& lay,
                                            bool shared_tab, const DecodeArgs& a, void* __restrict__ out,
                                            int64_t cimg, int gs, int ge, int gpi, float invW, float* stage,
                                            int warp, int lane, uint64_t* ready, uint32_t ready_phase) {
  using Net = NetView<HID, NL>;
  constexpr int GPX = NB * 16;
  constexpr int64_t GSTEP = M::STORE == 3 ? 3 * GPX : GPX;  // store offset advance per group (NHWC: x3)
  const StoreLane SL = make_store_lane<NB, M::STORE>(a, lane);
  // each warp takes a contiguous run of groups (few image changes per warp)
  const int cnt = ge - gs;
  const int w0g = gs + int((int64_t(cnt) * warp) / NW), w1g = gs + int((int64_t(cnt) * (warp + 1)) / NW);
  int i = w0g / gpi, within = w0g - i * gpi;
  int cur = -1;
  ImgRegs<HID, NL> R;
  R.set_norm(a, lane);
  Net net(const_cast<uint32_t*>(nets));
  int64_t obase = 0, gofs = 0;
  const float* colx = tabs;
  const float* rowy = tabs;
  SepRegs S;
  float* rowt = stage + 3 * GPX;  // [2][32] row-term buffers (SEP)
  if constexpr (M::SEP) {
    // out_w == GPX: group `within` is output row `within`.  Outer loop: one
    // image's run of rows (setup once); inner loop: straight rows, the next
    // row's terms computed one group ahead into the other row-term buffer.
    S.slot = sep_row_slot(lane);
    int gg = w0g;
#pragma unroll 1
    while (gg < w1g) {
      const int rows = min(gpi - within, w1g - gg);
      bulk_mbar_wait(&ready[i], ready_phase);  // image i's network is dequantised
      net = Net(const_cast<uint32_t*>(nets) + i * lay.net_words);
      R.load(net, lane);
      obase = (cimg + i) * 3 * int64_t(a.hw);
      gofs = obase + SL.goff + int64_t(within) * GSTEP;
      colx = shared_tab ? tabs : tabs + i * lay.tab_floats;
      rowy = colx + ((a.out_w + 3) & ~3);
      {
        const int g = lane >> 2, tq = lane & 3;
        const float4 lr = reinterpret_cast<const float4*>(net.l0)[lane & 15];
        S.w1 = lr.y;
        S.b1 = (lane >> 4) ? lr.z + 1.57079632679489662f : lr.z;  // cosine lanes: sin(r + pi/2)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float w0 = net.l0[4 * (2 * tq + (q & 1) + 8 * (q >> 1))];
#pragma unroll
          for (int bk = 0; bk < 2; ++bk)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float ax = w0 * colx[16 * bk + 8 * h + g];
              S.sa[bk][h][q] = __sinf(ax);
              S.ca[bk][h][q] = __cosf(ax);
            }
        }
      }
      float* rc = rowt;
      float* rn = rowt + 32;
      sep_row_terms(S, rowy[within], rc, S.slot);
      __syncwarp();
      const int rend = within + rows;
      // direct NCHW f32 stores: a running output pointer (no per-group address arithmetic)
      constexpr bool PTR = M::STORE == 1 && DIRECT_STORE1;
      float* op = static_cast<float*>(out) + (PTR ? gofs : 0);
      // the last row's look-ahead term (rowy[out_h]) is computed and unused
      auto row = [&](int r, float* cur, float* nxt) {
        decode_group<HID, NL, X3, ACCURATE, NB, M>(net, R, colx, rowy, a, PTR ? op : out, cimg + i, obase, r * GPX,
                                                   r, 0, stage, SL, lane, S, cur, nxt, true, PTR ? 0 : gofs);
        if constexpr (PTR) op += GSTEP;
        else gofs += GSTEP;
      };
      // two rows per trip: the row-term buffers alternate at compile time and
      // the compiler overlaps one row's epilogue with the next row's layer 0
      // (+2% over one row per trip)
      int r = within;
#pragma unroll 1
      for (; r + 1 < rend; r += 2) {
        row(r, rc, rn);
        row(r + 1, rn, rc);
      }
      if (r < rend) row(r, rc, rn);
      gg += rows;
      within = 0;
      ++i;
    }
  } else {
    int rb = (within * GPX) / a.out_w, cb = within * GPX - rb * a.out_w;
#pragma unroll 1
    for (int gg = w0g; gg < w1g; ++gg) {
      if (i != cur) {
        cur = i;
        bulk_mbar_wait(&ready[i], ready_phase);  // image i's network is dequantised
        net = Net(const_cast<uint32_t*>(nets) + i * lay.net_words);
        R.load(net, lane);
        obase = (cimg + i) * 3 * int64_t(a.hw);
        gofs = obase + SL.goff + int64_t(within) * GSTEP;
        colx = shared_tab ? tabs : tabs + i * lay.tab_floats;
        rowy = colx + ((a.out_w + 3) & ~3);
      }
      decode_group<HID, NL, X3, ACCURATE, NB, M>(net, R, colx, rowy, a, out, cimg + i, obase, within * GPX, rb, cb,
                                                 stage, SL, lane, S, rowt, rowt, false, gofs);
      gofs += GSTEP;
      cb += GPX;
      while (cb >= a.out_w) {
        cb -= a.out_w;
        ++rb;
      }
      if (++within == gpi) {
        within = 0;
        rb = 0;
        cb = 0;
        ++i;
      }
    }
  }
}

template <int HID, int NL, bool X3, bool ACCURATE, int NW, int NB, class M>
__global__ void __launch_bounds__(NW * 32, (NW < 16 ? 16 / NW : 1))
    decode_persist(StoreView sv, const int64_t* __restrict__ ids, int64_t n, DecodeArgs a,
                   const float* __restrict__ aug, void* __restrict__ out, int32_t* status, float omega,
                   PersistLayout lay, int overlap) {
  using C = MmaCfg<HID, NL>;
  using Net = NetView<HID, NL>;
  constexpr int NT = NW * 32;
  // Without the overlap promise the inputs may come from the preceding kernel:
  // wait for it before reading anything.
  if (!(overlap & 1)) pdl_wait();
  constexpr int GPX = NB * 16;
  // per-image parameter count in the flattened dequant walk (weights + biases)
  constexpr int P0 = 2 * HID + HID, PH = HID * HID + HID, PO = 3 * HID + 3;
  constexpr int PALL = P0 + (NL - 2) * PH + PO;
  constexpr int KW = (HID * HID + 31) / 32 + 1;  // words of one layer's bitset/prefix table
  // fragment-owner dequant tasks need every layer's bitset in one warp's registers
  constexpr bool FRAG_TASKS = HID <= 32;

  extern __shared__ __align__(16) uint8_t smem[];
  const bool shared_tab = a.aug == RINR_AUG_NONE;
  uint32_t* nets = reinterpret_cast<uint32_t*>(smem);
  float* tabs = reinterpret_cast<float*>(nets + lay.maxi * lay.net_words);
  uint8_t* recs = reinterpret_cast<uint8_t*>(tabs + (shared_tab ? 1 : lay.maxi) * lay.tab_floats);
  uint32_t* pfx = reinterpret_cast<uint32_t*>(recs + size_t(lay.maxi) * lay.rec_bytes);
  int64_t* metaid = reinterpret_cast<int64_t*>(pfx + lay.maxi * lay.pfx_words);  // [maxi]
  uint64_t* ready = reinterpret_cast<uint64_t*>(metaid + ((lay.maxi + 1) & ~1));   // [maxi] mbarriers
  float* stagebase = reinterpret_cast<float*>(ready + ((lay.maxi + 1) & ~1));

  dev_stamp(overlap, 0);
#ifdef RINR_DEV_KNOBS
  if (NW <= 8 && threadIdx.x == 0 && blockIdx.x < 512) {  // SM id in the unused warp-15 task slot
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_dev_task[blockIdx.x][15][0] = smid;
  }
#endif
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nblk = (a.hw + 15) / 16;
  const int gpi = (nblk + NB - 1) / NB;  // groups per image
  // CTA group range [G0, G1): 32-bit arithmetic (the launcher guarantees
  // n * gpi < 2^31; 64-bit divisions here cost ~60 instructions each)
  const uint32_t total = uint32_t(n) * uint32_t(gpi);
  const uint32_t qg = total / gridDim.x, rg = total - qg * gridDim.x;
  const uint32_t G0u = blockIdx.x * qg + min(blockIdx.x, rg);
  const uint32_t G1u = G0u + qg + (blockIdx.x < rg ? 1u : 0u);
  const int64_t G0 = G0u, G1 = G1u;
  if (G0u >= G1u) return;
  if (overlap & 8) {  // RINR_DEBUG_SKIP=4 (development builds): launch + PDL chain only
    pdl_wait();
    pdl_trigger();
    return;
  }
  const int64_t img0 = G0u / uint32_t(gpi);
  const int nimg = int((G1u - 1) / uint32_t(gpi) - uint32_t(img0) + 1);
  float* stage = stagebase + warp * (3 * GPX + 64);  // output stage + SEP row terms
  const float invW = 1.0f / float(a.out_w);
  // the first id of this warp is loaded before the setup below (its HBM
  // latency overlaps the table build and the barrier)
  const int64_t id_first = warp < min(lay.maxi, nimg) ? ids[img0 + warp] : 0;
  // RINR_FLAG_PREFETCH_NEXT (bit 64): ids[n, 2n) is the next batch; the same
  // grid split gives this CTA the same image range there, so each warp loads
  // one next-batch id now and prefetches its record slot into L2 after
  // phase 1 (the id load has landed by then; the next launch's record copies
  // then hit L2)
  const int64_t id_next = ((overlap & 64) && warp < nimg) ? ids[int64_t(n) + img0 + warp] : -1;
  // TMA bulk record copies: one mbarrier per warp (the warp that fetches a
  // record initialises, expects and arrives on its own barrier, so it needs
  // no CTA barrier before issuing); chunk k completes phase parity k & 1
  __shared__ uint64_t rec_mbar[NW];
  uint32_t rec_phase = 0;
  if (lane == 0) bulk_mbar_init(&rec_mbar[warp]);
  __syncwarp();
  // per-image readiness barriers, initialised once; chunk k waits on phase
  // parity k & 1 (every image slot of a chunk receives TASKS arrivals)
  constexpr uint32_t TASKS = FRAG_TASKS ? 1 + C::NH : NL;  // fragment-owner tasks or one per layer
  for (int i = tid; i < lay.maxi; i += NT) ready_init(&ready[i], TASKS);
  uint32_t ready_phase = 0;
  if (shared_tab) build_coord_tables(a, aug, 0, tabs, tabs + ((a.out_w + 3) & ~3), tid, NT);
  // (no barrier here: the in-chunk barrier below orders the tables and the
  // readiness barriers before any use)

  for (int c0 = 0; c0 < nimg; c0 += lay.maxi) {
    const int ni = min(lay.maxi, nimg - c0);
    const int64_t cimg = img0 + c0;  // first image of the chunk
    // -------------------------------- phase 1 --------------------------------
    // Slot copies: warp w fetches the ids of images w, w+NW, ... and streams
    // their slots into shared memory (one dependent load: the id).
    for (int i = warp; i < ni; i += NW) {
      const int64_t id = (c0 == 0 && i == warp) ? id_first : ids[cimg + i];
      const bool ok = id >= 0 && id < sv.n;
      if (c0 == 0 && i == 0 && ok) dev_stamp(overlap, 7);
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
      if (lane == 0) bulk_copy_g2s(dst, src, bytes, &rec_mbar[warp]);  // one TMA bulk copy per record
    }
    if (lane == 0) bulk_mbar_arrive(&rec_mbar[warp]);  // after this warp's expect_tx of the chunk
    if (c0 == 0) dev_stamp(overlap, 1);
    if constexpr (!FRAG_TASKS)
      for (int i = tid; i < ni * lay.net_words / 4; i += NT) reinterpret_cast<uint4*>(nets)[i] = make_uint4(0, 0, 0, 0);
    if (!shared_tab)
      for (int i = 0; i < ni; ++i) {
        float* tab = tabs + i * lay.tab_floats;
        build_coord_tables(a, aug, cimg + i, tab, tab + ((a.out_w + 3) & ~3), tid, NT);
      }
    __syncthreads();  // metaid / tables / readiness barriers visible to every warp
    if (c0 == 0) dev_stamp(overlap, 2);
    // Dequantise straight into MMA fragments: task (image i, part h) with
    // h = 0 -> layer 0 + output layer, h = 1..NH -> hidden layer h.  Every
    // lane writes exactly the fragment words it owns (padding included), so
    // the network image needs no zero fill.
    if constexpr (FRAG_TASKS) {
      constexpr int TPI = 1 + C::NH;
      for (int task = (overlap & 4) ? ni * TPI : warp; task < ni * TPI; task += NW) {
        const int i = task / TPI, h = task - i * TPI;
        if (metaid[i] >= 0) {
          bulk_mbar_wait(&rec_mbar[i % NW], rec_phase);  // record i is in shared memory
#ifdef RINR_DEV_KNOBS
          const unsigned long long t_a = clock64();
#endif
          frag_task<HID, NL, M::INTB>(sv, recs + size_t(i) * lay.rec_bytes, h, Net(nets + i * lay.net_words), omega,
                                      lane);
#ifdef RINR_DEV_KNOBS
          __syncwarp();
          if (lane == 0 && blockIdx.x < 512 && warp < 16 && task == warp) {
            g_dev_task[blockIdx.x][warp][0] = t_a;
            g_dev_task[blockIdx.x][warp][1] = clock64() - t_a + 1000000ull * h;
          }
#endif
        }
        __syncwarp();  // the warp's fragment writes happen before lane 0's release
        if (lane == 0) ready_arrive(&ready[i]);
      }
    }
    // Dequantise: one warp per (image, layer) task — the layer header is parsed
    // once, the kept-bit prefix table is built by the same warp, then the
    // lanes stride over the layer's weights and biases.
    if constexpr (!FRAG_TASKS)
    for (int task = (overlap & 4) ? ni * NL : warp; task < ni * NL; task += NW) {
      const int i = task / NL, l = task - i * NL;
      if (metaid[i] < 0) {
        if (lane == 0) ready_arrive(&ready[i]);
        continue;
      }
      bulk_mbar_wait(&rec_mbar[i % NW], rec_phase);  // record i is in shared memory
      const uint32_t* lo = reinterpret_cast<const uint32_t*>(recs + size_t(i) * lay.rec_bytes);
      const uint8_t* rec = recs + size_t(i) * lay.rec_bytes + sv.hdr_bytes;
      const int fi = l == 0 ? 2 : HID, fo = l == NL - 1 ? 3 : HID;
      const DLayer L = parse_layer(rec, lo[l], lo[l + 1], fi, fo);
      uint32_t* words = pfx + i * lay.pfx_words + l * 2 * KW;
      if (L.form != FORM_DENSE) {
        build_bit_prefix(rec, L, words, words + KW, lane);
        __syncwarp();
      }
      const bool hidden = l > 0 && l < NL - 1;
      const bool int_b = hidden && int_b_exact(L);
      Net net(nets + i * lay.net_words);
      if (l == 0) {
        for (int j = lane; j < L.n; j += 32)
          net.l0[(j >> 1) * 4 + (j & 1)] = __fmul_rn(omega, dq_weight(rec, L, words, words + KW, j));
        for (int o = lane; o < fo; o += 32) net.l0[o * 4 + 2] = __fmul_rn(omega, dq_bias(rec, L, o));
      } else if (hidden) {
        uint32_t* fr = net.fragH + (l - 1) * C::KT * C::NT * 32 * 4;
        if (int_b) {
          for (int j = lane; j < L.n; j += 32) {
            const int o = j / HID, k = j - o * HID;
            Net::put_b(fr, C::NT, k, o, dq_int(rec, L, words, words + KW, j), 0.0f);
          }
        } else {
          for (int j = lane; j < L.n; j += 32) {
            const int o = j / HID, k = j - o * HID;
            Net::put_b_split(fr, C::NT, k, o, __fmul_rn(omega, dq_weight(rec, L, words, words + KW, j)));
          }
        }
        for (int o = lane; o < fo; o += 32) net.biasH[(l - 1) * C::NT * 8 + o] = __fmul_rn(omega, dq_bias(rec, L, o));
        if (lane == 0) {
          net.modeH[l - 1] = int_b ? 1 : 0;
          net.scaleH[l - 1] = int_b ? __double2float_rn(double(omega) * L.scale) : 1.0f;
        }
      } else {
        for (int j = lane; j < L.n; j += 32) {
          const int o = j / HID, k = j - o * HID;
          Net::put_b_split(net.fragO, 1, k, 2 * o, dq_weight(rec, L, words, words + KW, j));  // column 2o
        }
        for (int o = lane; o < fo; o += 32) net.biasO[o] = dq_bias(rec, L, o);
      }
      __syncwarp();  // the warp's writes happen before lane 0's release
      if (lane == 0) ready_arrive(&ready[i]);
    }
    if (overlap & 4) {  // RINR_DEBUG_SKIP=1 (development builds): no dequant tasks ran
      if (tid < ni)
        for (uint32_t k = 0; k < TASKS; ++k) ready_arrive(&ready[tid]);
    }
    // -------------------------------- phase 2 --------------------------------
    // No CTA barrier here: each warp starts its groups as soon as the
    // networks of its images are ready (phase2_loop waits on `ready`).
    if (c0 == 0) {
      if (tid == 0) dev_stamp(overlap, 3);
      if (overlap & 1) pdl_wait();  // outputs may still be read/written by the preceding grid
      pdl_trigger();            // every CTA is resident: the next launch may start its prologue
      if (tid == 0) dev_stamp(overlap, 4);
      if (lane == 0 && id_next >= 0 && id_next < sv.n) {
        uint64_t off;
        uint32_t bytes;
        slot_of(sv, id_next, off, bytes);
        bulk_prefetch_l2(sv.blob + off, bytes);
      }
    }
    const int64_t cbase = cimg * gpi;
    const int gs = int((G0 > cbase ? G0 : cbase) - cbase);
    const int ge = int((G1 < cbase + int64_t(ni) * gpi ? G1 : cbase + int64_t(ni) * gpi) - cbase);
    if (!(overlap & 2))
      phase2_loop<HID, NL, X3, ACCURATE, NW, NB, M>(nets, tabs, lay, shared_tab, a, out, cimg, gs, ge, gpi, invW,
                                                    stage, warp, lane, ready, ready_phase);
    if (c0 == 0) dev_stamp(overlap, 5);
    ready_phase ^= 1u;
    rec_phase ^= 1u;
    __syncthreads();
  }
  dev_stamp(overlap, 6);
}

}  // namespace rinr
