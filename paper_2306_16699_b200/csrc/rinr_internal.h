// Internal declarations shared by the host store builder (store.cpp) and the
// CUDA kernels (decode.cu).  Not part of the ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/rinr_b200.h"

namespace rinr {

// .rinr constants (reference archive.py:45-58).
constexpr uint8_t TAG_F32 = 0, TAG_F16 = 1, TAG_A8 = 2, TAG_A16 = 3;
constexpr uint8_t FORM_DENSE = 0, FORM_DENSE_MASK = 1, FORM_SPARSE = 2;

constexpr int kMaxDims = 32;          // widths per architecture (incl. in/out)
constexpr int kRecordAlign = 16;      // every record starts 16-B aligned in HBM
constexpr int kBlobTailPad = 64;      // over-read slack after the last record

// Device-side view of an immutable store.  Passed by value to kernels.
//
// HBM layout (one allocation):
//   blob     : one 16-B aligned slot per record:
//                [u32 layer offsets x lstride, zero padded to hdr_bytes]
//                [record body (id .. last bias; CRC stripped), padded to 16 B]
//              Layer offset l is the position of layer l's tag byte relative
//              to the body start; entry [n_layers] is the end of the body, so
//              the bias of layer l sits at off[l+1] - 4*out_l.  A whole slot
//              moves with 16-B vector loads / cp.async.  When record sizes are
//              close (always, for a homogeneous dataset) every slot has the
//              same size `slot_stride` and slot k starts at k * slot_stride,
//              so a kernel reaches a record with a single dependent load (the
//              id); otherwise slot_stride = 0 and rec_off[k]..rec_off[k+1]
//              bound slot k.  kBlobTailPad zero bytes follow the last slot.
//   rec_off  : u64 [n + 1]      slot boundaries
//   arch_idx : u16 [n]          index into the architecture table
//   arch_dims: u16 [n_arch * kMaxDims], arch_nd: i32 [n_arch],
//   arch_omega: f32 [n_arch]    f32(omega) as the reference's forward uses it
//                               (net.py:200 under NEP 50)
struct StoreView {
  const uint8_t* blob;
  const uint64_t* rec_off;
  const uint16_t* arch_idx;
  const uint16_t* arch_dims;
  const int32_t* arch_nd;
  const float* arch_omega;
  int64_t n;
  int32_t lstride;          // layer-offset entries per slot header (max layers + 1)
  int32_t hdr_bytes;        // slot header size (16-B multiple)
  int64_t slot_stride;      // fixed slot size, or 0 for variable slots
  int32_t n_arch;
  int32_t max_slot_bytes;   // largest slot (16-B multiple)
  int32_t max_params;
  int32_t max_width;
  int32_t hidden_int8;      // 1: every hidden layer of every record is affine8 codes
};

// Slot of record `id`: start and size in bytes.
#ifdef __CUDACC__
__device__ __forceinline__ void slot_of(const StoreView& sv, int64_t id, uint64_t& off, uint32_t& bytes) {
  if (sv.slot_stride) {
    off = uint64_t(id) * uint64_t(sv.slot_stride);
    bytes = uint32_t(sv.slot_stride);
  } else {
    off = sv.rec_off[id];
    bytes = uint32_t(sv.rec_off[id + 1] - off);
  }
}
#endif

struct HostArch {
  int nd;
  uint16_t dims[kMaxDims];
  double omega;
};

// Thread-local error helpers (capi.cpp).
int set_error(int code, const std::string& msg, int64_t record = -1);
void clear_error();

}  // namespace rinr

// Kernel launchers (decode.cu).  Return RINR_OK or an error code (message set).
int rinr_launch_dequantize(const rinr::StoreView& sv, const int64_t* d_ids, int64_t n,
                           float* d_out, int64_t out_stride, int32_t* d_status, void* stream);
int rinr_launch_decode(const rinr::StoreView& sv, const rinr::HostArch* uniform_arch,
                       const int64_t* d_ids, int64_t n, const rinr_decode_params_t* p,
                       const float* d_aug, void* d_out, int32_t* d_status, void* stream);
