// GPU .rinr writer ("GPU-side synthetic generator"):
// serialises a device-resident batch of same-architecture models (the
// transform layout of rinr_b200_transforms.h plus the quantize results)
// straight into archive bytes in device memory, byte-identical to the
// reference writer (archive.py:92-184: _layer_plan, _encode_layer,
// encode_record, serialize) and to the host writer (archive.py here).
//
//   ser_size_kernel   one warp per record: kept counts -> per-layer form and
//                     the record length (archive.py:100-108, 132-135)
//   (host)            exclusive scan of the lengths -> record offsets
//   ser_write_kernel  one warp per record: every field, byte by byte; index
//                     entry; the archive header (record 0's warp)
//   ser_crc_kernel    one thread per record: zlib CRC-32 of the body, table
//                     in shared memory (archive.py:9-24)
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/rinr_b200_writer.h"
#include "rinr_internal.h"

namespace rinr {
namespace {

constexpr int kWMaxLayers = 31;
constexpr int kIdMax = 48;

struct WArch {
  int nl, nd, P;
  int dims[kWMaxLayers + 1];
  int off[kWMaxLayers + 1];   // weight offset of matrix l
  int boff[kWMaxLayers + 1];  // bias offset of layer l
  int bsum;                   // biases per model
};

struct WCfg {
  WArch A;
  int quant_bits;        // 0 = none, 8, 16
  uint32_t src_h, src_w;
  double omega;
  int64_t first_id;
  int id_width;
  int prefix_len;
  char prefix[kIdMax];
};

__device__ __forceinline__ bool is_quant(const WCfg& c, int l) { return c.quant_bits && l > 0 && l + 1 < c.A.nl; }

// Decimal id of record i: prefix + zero-padded index (Python f"{prefix}{i:0{w}d}").
__device__ __forceinline__ int id_digits(int64_t v, int width) {
  int d = 1;
  for (int64_t t = v; t >= 10; t /= 10) ++d;
  return d > width ? d : width;
}

__global__ void ser_size_kernel(WCfg c, int64_t n, const uint8_t* __restrict__ mask, const uint8_t* __restrict__ cst,
                                uint8_t* __restrict__ forms, int32_t* __restrict__ kept, int64_t* __restrict__ rec_len) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  const WArch& A = c.A;
  const uint8_t* m = mask + r * A.P;
  const int nh = A.nl - 2;
  int64_t len = 2 + c.prefix_len + id_digits(c.first_id + r, c.id_width) + 8 + 2 + 2 * A.nd + 8 + 1;
  for (int l = 0; l < A.nl; ++l) {
    const int size = A.dims[l] * A.dims[l + 1];
    int cnt = 0;
    for (int j = lane; j < size; j += 32) cnt += m[A.off[l] + j] != 0;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    const int zeros = size - cnt;
    // dense if no zeros, sparse if zeros / size > 1/8, else dense + bitset
    const int form = zeros == 0 ? 0 : (8 * zeros > size ? 2 : 1);
    const bool q = is_quant(c, l);
    const bool cq = q && nh > 0 && cst[r * nh + (l - 1)];
    const int isz = q && !cq ? c.quant_bits / 8 : 4;
    const int nvals = form == 2 ? cnt : size;
    len += 3 + (q ? 12 : 0) + (form ? (size + 7) / 8 : 0) + int64_t(nvals) * isz + 4 * A.dims[l + 1];
    if (lane == 0) {
      forms[r * A.nl + l] = uint8_t(form);
      kept[r * A.nl + l] = cnt;
    }
  }
  if (lane == 0) rec_len[r] = len + 4;  // + CRC
}

struct ByteOut {
  uint8_t* p;
  __device__ __forceinline__ void put(int64_t o, uint8_t v) const { p[o] = v; }
  template <class T>
  __device__ __forceinline__ void put_le(int64_t o, T v) const {
    uint64_t u = 0;
    memcpy(&u, &v, sizeof(T));
#pragma unroll
    for (int k = 0; k < int(sizeof(T)); ++k) p[o + k] = uint8_t(u >> (8 * k));
  }
};

__global__ void ser_write_kernel(WCfg c, int64_t n, const float* __restrict__ w, const uint8_t* __restrict__ mask,
                                 const float* __restrict__ b, const double* __restrict__ scale,
                                 const int32_t* __restrict__ zp, const uint8_t* __restrict__ cst,
                                 const uint16_t* __restrict__ codes, const uint8_t* __restrict__ forms,
                                 const int32_t* __restrict__ kept, const int64_t* __restrict__ rec_off,
                                 const int64_t* __restrict__ rec_len, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  const WArch& A = c.A;
  const ByteOut o{out};
  const int64_t hdr = 10 + 12 * n;
  if (r == 0 && lane == 0) {  // "<4sHI": magic, version 1, count
    o.put(0, 'R'); o.put(1, 'I'); o.put(2, 'N'); o.put(3, 'R');
    o.put_le<uint16_t>(4, 1);
    o.put_le<uint32_t>(6, uint32_t(n));
  }
  int64_t p = hdr + rec_off[r];
  if (lane == 0) {  // index entry "<QI": offset, length
    o.put_le<uint64_t>(10 + 12 * r, uint64_t(p));
    o.put_le<uint32_t>(10 + 12 * r + 8, uint32_t(rec_len[r]));
  }
  // id, source size, architecture, omega, quant mode (archive.py:140-158)
  const int64_t idv = c.first_id + r;
  const int nd = id_digits(idv, c.id_width);
  const int id_len = c.prefix_len + nd;
  if (lane == 0) {
    o.put_le<uint16_t>(p, uint16_t(id_len));
    for (int k = 0; k < c.prefix_len; ++k) o.put(p + 2 + k, uint8_t(c.prefix[k]));
    int64_t t = idv;
    for (int k = nd - 1; k >= 0; --k) {
      o.put(p + 2 + c.prefix_len + k, uint8_t('0' + t % 10));
      t /= 10;
    }
  }
  p += 2 + id_len;
  if (lane == 0) {
    o.put_le<uint32_t>(p, c.src_h);
    o.put_le<uint32_t>(p + 4, c.src_w);
    o.put_le<uint16_t>(p + 8, uint16_t(A.nd));
    for (int k = 0; k < A.nd; ++k) o.put_le<uint16_t>(p + 10 + 2 * k, uint16_t(A.dims[k]));
    o.put_le<double>(p + 10 + 2 * A.nd, c.omega);
    o.put(p + 18 + 2 * A.nd, uint8_t(c.quant_bits == 0 ? 0 : (c.quant_bits == 8 ? 1 : 2)));
  }
  p += 19 + 2 * A.nd;
  const int nh = A.nl - 2;
  for (int l = 0; l < A.nl; ++l) {
    const int fi = A.dims[l], fo = A.dims[l + 1], size = fi * fo;
    const int form = forms[r * A.nl + l];
    const bool q = is_quant(c, l);
    const bool cq = q && cst[r * nh + (l - 1)];
    if (lane == 0) {
      o.put(p, uint8_t(q ? (c.quant_bits == 8 ? 2 : 3) : 0));  // tag: f32 / affine8 / affine16
      o.put(p + 1, uint8_t(form));
      o.put(p + 2, uint8_t(cq ? 1 : 0));
      if (q) {
        o.put_le<double>(p + 3, scale[r * nh + (l - 1)]);
        o.put_le<int32_t>(p + 11, zp[r * nh + (l - 1)]);
      }
    }
    p += 3 + (q ? 12 : 0);
    const uint8_t* m = mask + r * A.P + A.off[l];
    if (form) {  // kept bitset, LSB first (np.packbits bitorder="little")
      const int nb = (size + 7) / 8;
      for (int k = lane; k < nb; k += 32) {
        uint8_t v = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (8 * k + t < size && m[8 * k + t]) v |= uint8_t(1u << t);
        o.put(p + k, v);
      }
      p += nb;
    }
    // values: every entry (dense forms) or the kept ones in order (sparse)
    const int isz = q && !cq ? c.quant_bits / 8 : 4;
    const float* wl = w + r * A.P + A.off[l];
    const uint16_t* cl = codes + r * A.P + A.off[l];
    int base = 0;
    for (int j0 = 0; j0 < size; j0 += 32) {
      const int j = j0 + lane;
      const bool in = j < size;
      const bool sel = in && (form != 2 || m[j] != 0);
      const uint32_t bal = __ballot_sync(0xffffffffu, sel);
      if (sel) {
        const int64_t at = p + int64_t(base + __popc(bal & ((1u << lane) - 1u))) * isz;
        if (isz == 1) o.put(at, uint8_t(cl[j]));
        else if (isz == 2) o.put_le<uint16_t>(at, cl[j]);
        else o.put_le<float>(at, wl[j]);
      }
      base += __popc(bal);
    }
    p += int64_t(base) * isz;
    for (int k = lane; k < fo; k += 32) o.put_le<float>(p + 4 * k, b[r * A.bsum + A.boff[l] + k]);
    p += 4 * fo;
  }
}

__device__ uint32_t crc_table_entry(uint32_t i) {
  uint32_t c = i;
  for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
  return c;
}

__global__ void __launch_bounds__(256) ser_crc_kernel(int64_t n, const int64_t* __restrict__ rec_off,
                                                     const int64_t* __restrict__ rec_len, uint8_t* __restrict__ out) {
  __shared__ uint32_t table[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) table[i] = crc_table_entry(uint32_t(i));
  __syncthreads();
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int64_t start = 10 + 12 * n + rec_off[r], body = rec_len[r] - 4;
  const uint8_t* p = out + start;
  uint32_t crc = 0xFFFFFFFFu;
  for (int64_t k = 0; k < body; ++k) crc = table[(crc ^ p[k]) & 0xFFu] ^ (crc >> 8);
  crc = ~crc;
  uint8_t* t = out + start + body;
#pragma unroll
  for (int k = 0; k < 4; ++k) t[k] = uint8_t(crc >> (8 * k));
}

int warch_of(const int32_t* dims, int nl, WArch& A) {
  if (!dims || nl < 1 || nl > kWMaxLayers) return set_error(RINR_ERR_INVALID_INPUT, "bad layer count");
  A.nl = nl;
  A.nd = nl + 1;
  A.P = 0;
  A.bsum = 0;
  for (int l = 0; l <= nl; ++l) {
    if (dims[l] < 1 || dims[l] > 0xFFFF) return set_error(RINR_ERR_INVALID_INPUT, "layer width out of range");
    A.dims[l] = dims[l];
  }
  if (dims[0] != 2 || dims[nl] != 3) return set_error(RINR_ERR_INVALID_INPUT, "architecture must map 2 -> 3");
  for (int l = 0; l < nl; ++l) {
    A.off[l] = A.P;
    A.boff[l] = A.bsum;
    A.P += dims[l] * dims[l + 1];
    A.bsum += dims[l + 1];
  }
  return RINR_OK;
}

}  // namespace
}  // namespace rinr

using namespace rinr;

extern "C" int rinr_serialize_size(const rinr_serialize_args_t* a, int64_t* d_rec_len, uint8_t* d_forms,
                                   int32_t* d_kept, void* stream) {
  clear_error();
  if (!a) return set_error(RINR_ERR_INVALID_INPUT, "null args");
  WCfg c{};
  if (int e = warch_of(a->dims, a->n_layers, c.A)) return e;
  if (a->n < 0) return set_error(RINR_ERR_INVALID_INPUT, "negative n");
  if (a->quant_bits != 0 && a->quant_bits != 8 && a->quant_bits != 16)
    return set_error(RINR_ERR_INVALID_INPUT, "quant_bits must be 0, 8 or 16");
  if (a->n == 0) return RINR_OK;
  if (!a->d_mask || !d_rec_len || !d_forms || !d_kept || (a->quant_bits && c.A.nl > 2 && !a->d_const))
    return set_error(RINR_ERR_INVALID_INPUT, "null buffer");
  const int plen = a->id_prefix ? int(strnlen(a->id_prefix, kIdMax)) : 0;
  if (plen >= kIdMax) return set_error(RINR_ERR_INVALID_INPUT, "id prefix too long");
  c.quant_bits = a->quant_bits;
  c.first_id = a->first_id;
  c.id_width = a->id_width;
  c.prefix_len = plen;
  const int64_t threads = a->n * 32;
  ser_size_kernel<<<unsigned((threads + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      c, a->n, a->d_mask, a->d_const, d_forms, d_kept, d_rec_len);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RINR_OK : set_error(RINR_ERR_CUDA, std::string("serialize size: ") + cudaGetErrorString(e));
}

extern "C" int rinr_serialize_write(const rinr_serialize_args_t* a, const int64_t* d_rec_off, const int64_t* d_rec_len,
                                    const uint8_t* d_forms, const int32_t* d_kept, uint8_t* d_out, void* stream) {
  clear_error();
  if (!a) return set_error(RINR_ERR_INVALID_INPUT, "null args");
  WCfg c{};
  if (int e = warch_of(a->dims, a->n_layers, c.A)) return e;
  if (a->n < 0) return set_error(RINR_ERR_INVALID_INPUT, "negative n");
  if (a->quant_bits != 0 && a->quant_bits != 8 && a->quant_bits != 16)
    return set_error(RINR_ERR_INVALID_INPUT, "quant_bits must be 0, 8 or 16");
  const bool hq = a->quant_bits && c.A.nl > 2;
  if (!d_out || (a->n && (!a->d_w || !a->d_mask || !a->d_b || !d_rec_off || !d_rec_len || !d_forms || !d_kept ||
                          (hq && (!a->d_scale || !a->d_zp || !a->d_const || !a->d_codes)))))
    return set_error(RINR_ERR_INVALID_INPUT, "null buffer");
  const int plen = a->id_prefix ? int(strnlen(a->id_prefix, kIdMax)) : 0;
  if (plen >= kIdMax) return set_error(RINR_ERR_INVALID_INPUT, "id prefix too long");
  c.quant_bits = a->quant_bits;
  c.src_h = a->source_h;
  c.src_w = a->source_w;
  c.omega = a->omega;
  c.first_id = a->first_id;
  c.id_width = a->id_width;
  c.prefix_len = plen;
  for (int k = 0; k < plen; ++k) c.prefix[k] = a->id_prefix[k];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a->n == 0) {  // header only
    const uint8_t h[10] = {'R', 'I', 'N', 'R', 1, 0, 0, 0, 0, 0};
    const cudaError_t e = cudaMemcpyAsync(d_out, h, 10, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) cudaStreamSynchronize(st);  // h lives on this stack frame
    return e == cudaSuccess ? RINR_OK : set_error(RINR_ERR_CUDA, "serialize header copy");
  }
  const int64_t threads = a->n * 32;
  ser_write_kernel<<<unsigned((threads + 255) / 256), 256, 0, st>>>(c, a->n, a->d_w, a->d_mask, a->d_b, a->d_scale,
                                                                    a->d_zp, a->d_const, a->d_codes, d_forms, d_kept,
                                                                    d_rec_off, d_rec_len, d_out);
  ser_crc_kernel<<<unsigned((a->n + 255) / 256), 256, 0, st>>>(a->n, d_rec_off, d_rec_len, d_out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RINR_OK
                          : set_error(RINR_ERR_CUDA, std::string("serialize write: ") + cudaGetErrorString(e));
}
