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
// HBM layout (one allocation each):
//   blob     : record bodies (id .. last bias; CRC stripped), each starting at
//              a 16-B aligned offset so a whole record moves with 16-B vector
//              loads / one bulk copy; followed by kBlobTailPad zero bytes.
//   rec_off  : u64 [n]          byte offset of record k in blob
//   lay_off  : u32 [n * lstride] offset (from record start) of each layer's
//              tag byte; entry [n_layers] = end of the body.  The bias of layer
//              l therefore sits at lay_off[l+1] - 4*out_l.
//   arch_idx : u16 [n]          index into the architecture table
//   arch_dims: u16 [n_arch * kMaxDims], arch_nd: i32 [n_arch],
//   arch_omega: f32 [n_arch]    f32(omega) as the reference's forward uses it
//                               (net.py:200 under NEP 50)
struct StoreView {
  const uint8_t* blob;
  const uint64_t* rec_off;
  const uint32_t* lay_off;
  const uint16_t* arch_idx;
  const uint16_t* arch_dims;
  const int32_t* arch_nd;
  const float* arch_omega;
  int64_t n;
  int32_t lstride;
  int32_t n_arch;
  int32_t max_record_bytes;   // rounded up to 16
  int32_t max_params;
  int32_t max_width;
};

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
