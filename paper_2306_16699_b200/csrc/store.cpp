// Host side of the store: .rinr parsing/validation (mirrors reference
// archive.py:187-400), CRC32, the HBM upload, and the C-ABI entry points that
// are not kernels.  Pure C++ except for the CUDA runtime calls in
// rinr_store_create/destroy.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <memory>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "rinr_internal.h"

namespace rinr {

// ----------------------------------------------------------------------------
// errors (thread-local, like errno)
// ----------------------------------------------------------------------------
static thread_local std::string g_err;
static thread_local int64_t g_err_record = -1;

int set_error(int code, const std::string& msg, int64_t record) {
  g_err = msg;
  g_err_record = record;
  return code;
}
void clear_error() {
  g_err.clear();
  g_err_record = -1;
}

// ----------------------------------------------------------------------------
// CRC-32 (IEEE 802.3, reflected poly 0xEDB88320 — zlib.crc32, archive.py:158,
// 332), slicing-by-8.
// ----------------------------------------------------------------------------
static uint32_t g_crc_tab[8][256];
static bool g_crc_init = [] {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    g_crc_tab[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; ++i)
    for (int t = 1; t < 8; ++t) g_crc_tab[t][i] = (g_crc_tab[t - 1][i] >> 8) ^ g_crc_tab[0][g_crc_tab[t - 1][i] & 0xFF];
  return true;
}();

static uint32_t crc32(const uint8_t* p, size_t n) {
  uint32_t c = 0xFFFFFFFFu;
  while (n >= 8) {
    uint32_t lo, hi;
    std::memcpy(&lo, p, 4);
    std::memcpy(&hi, p + 4, 4);
    lo ^= c;
    c = g_crc_tab[7][lo & 0xFF] ^ g_crc_tab[6][(lo >> 8) & 0xFF] ^ g_crc_tab[5][(lo >> 16) & 0xFF] ^
        g_crc_tab[4][lo >> 24] ^ g_crc_tab[3][hi & 0xFF] ^ g_crc_tab[2][(hi >> 8) & 0xFF] ^
        g_crc_tab[1][(hi >> 16) & 0xFF] ^ g_crc_tab[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) c = g_crc_tab[0][(c ^ *p++) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// ----------------------------------------------------------------------------
// Parsing
// ----------------------------------------------------------------------------
struct ParseError {
  int code;
  std::string msg;
};

template <class T>
static T rd(const uint8_t* p) {
  T v;
  std::memcpy(&v, p, sizeof(T));
  return v;
}

struct ParsedRecord {
  bool hidden_int8 = true;   // every hidden layer stored as (non-constant) affine8 codes
  size_t body_off = 0;       // offset of the body in the archive image
  uint32_t body_len = 0;     // without CRC
  uint32_t source_h = 0, source_w = 0;
  HostArch arch{};
  std::vector<uint32_t> lay_off;  // n_layers + 1, relative to body start
  std::string id;
};

// Walk one record body (CRC already stripped).  Mirrors parse_record
// (archive.py:233-275): same field order, same failure cases, same messages.
static void parse_body(const uint8_t* b, size_t len, const std::string& ctx, ParsedRecord& out) {
  size_t pos = 0;
  auto take = [&](size_t n) -> const uint8_t* {
    if (pos + n > len)
      throw ParseError{RINR_ERR_INTEGRITY,
                       ctx + ": truncated (needed " + std::to_string(n) + " bytes at " + std::to_string(pos) + ")"};
    const uint8_t* p = b + pos;
    pos += n;
    return p;
  };
  uint16_t id_len = rd<uint16_t>(take(2));
  const uint8_t* idp = take(id_len);
  out.id.assign(reinterpret_cast<const char*>(idp), id_len);
  out.source_h = rd<uint32_t>(take(4));
  out.source_w = rd<uint32_t>(take(4));
  uint16_t nd = rd<uint16_t>(take(2));
  const uint8_t* dp = take(size_t(2) * nd);
  double omega = rd<double>(take(8));
  // Architecture invariants (net.py:36-47) -> IntegrityError (archive.py:242-245)
  bool ok = nd >= 2;
  for (int i = 0; ok && i < nd; ++i) ok = rd<uint16_t>(dp + 2 * i) >= 1;
  if (!ok || rd<uint16_t>(dp) != 2 || rd<uint16_t>(dp + 2 * (nd - 1)) != 3 || !(omega > 0))
    throw ParseError{RINR_ERR_INTEGRITY, ctx + ": bad architecture"};
  if (nd > kMaxDims)
    throw ParseError{RINR_ERR_UNSUPPORTED, ctx + ": " + std::to_string(nd) + " widths exceed this build's limit of " +
                                               std::to_string(kMaxDims)};
  out.arch.nd = nd;
  for (int i = 0; i < nd; ++i) out.arch.dims[i] = rd<uint16_t>(dp + 2 * i);
  out.arch.omega = omega;
  uint8_t mode = *take(1);
  if (mode > 2) throw ParseError{RINR_ERR_INTEGRITY, ctx + ": unknown quant mode " + std::to_string(mode)};
  out.lay_off.assign(nd, 0);
  for (int l = 0; l + 1 < nd; ++l) {
    out.lay_off[l] = uint32_t(pos);
    size_t fan_in = out.arch.dims[l], fan_out = out.arch.dims[l + 1];
    size_t n = fan_in * fan_out;
    const uint8_t* h = take(3);
    uint8_t tag = h[0], form = h[1], cst = h[2];
    if (tag > TAG_A16 || form > FORM_SPARSE)
      throw ParseError{RINR_ERR_INTEGRITY, ctx + ": layer " + std::to_string(l) + " has bad tag/form " +
                                               std::to_string(tag) + "/" + std::to_string(form)};
    bool affine = tag == TAG_A8 || tag == TAG_A16;
    int32_t zp = 0;
    if (affine) zp = rd<int32_t>(take(12) + 8);
    // integer-B MMA operand only when every code - zp is exact in bf16
    // (device_common.cuh int_b_exact)
    if (l > 0 && l + 2 < nd && !(tag == TAG_A8 && !cst && zp >= -1 && zp <= 256)) out.hidden_int8 = false;
    size_t kept = n;
    if (form != FORM_DENSE) {
      const uint8_t* bits = take((n + 7) / 8);
      if (form == FORM_SPARSE) {
        kept = 0;
        for (size_t j = 0; j < n; ++j) kept += (bits[j >> 3] >> (j & 7)) & 1;
      }
    }
    // values: f32 when a const affine layer, else the tag's dtype (archive.py:266)
    size_t isz = (cst && affine) ? 4 : (tag == TAG_F32 ? 4 : tag == TAG_F16 ? 2 : tag == TAG_A8 ? 1 : 2);
    take(kept * isz);
    take(4 * fan_out);
  }
  if (pos != len)
    throw ParseError{RINR_ERR_INTEGRITY, ctx + ": " + std::to_string(len - pos) + " trailing bytes"};
  out.lay_off[nd - 1] = uint32_t(pos);
  out.body_len = uint32_t(len);
}

struct ParsedArchive {
  uint16_t version = 0;
  int64_t count = 0;
  std::vector<ParsedRecord> recs;  // only the selected shard
  std::vector<int64_t> global;     // global index of each kept record
};

// Header, chained index, CRC and parse of every record (ArchiveReader +
// read(), archive.py:338-400).  Every record is validated even when only a
// shard is kept, so a corrupt archive fails identically on every rank.
static void parse_archive(const uint8_t* data, size_t len, uint32_t rank, uint32_t world, ParsedArchive& pa,
                          bool keep) {
  if (len < 10) throw ParseError{RINR_ERR_INTEGRITY, "truncated header"};
  if (std::memcmp(data, "RINR", 4) != 0) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "bad magic b'%c%c%c%c'", data[0], data[1], data[2], data[3]);
    throw ParseError{RINR_ERR_INTEGRITY, buf};
  }
  pa.version = rd<uint16_t>(data + 4);
  if (pa.version > 1) throw ParseError{RINR_ERR_INTEGRITY, "unsupported version " + std::to_string(pa.version)};
  uint32_t count = rd<uint32_t>(data + 6);
  pa.count = count;
  if (len < 10 + size_t(12) * count) throw ParseError{RINR_ERR_INTEGRITY, "truncated index"};
  // Offset chain first, for every record (ArchiveReader.__init__, archive.py:357-364) ...
  uint64_t expect = 10 + uint64_t(12) * count;
  for (uint32_t k = 0; k < count; ++k) {
    uint64_t off = rd<uint64_t>(data + 10 + 12 * size_t(k));
    uint32_t length = rd<uint32_t>(data + 10 + 12 * size_t(k) + 8);
    if (off != expect)
      throw ParseError{RINR_ERR_INTEGRITY, "record " + std::to_string(k) + ": offset " + std::to_string(off) +
                                               " != expected " + std::to_string(expect)};
    expect = off + length;
  }
  // ... then each record's bytes, CRC and parse (read_raw, archive.py:369-379).
  // Records are independent, so contiguous ranges run on host threads; each
  // thread stops at its first failure and the lowest-index failure is raised,
  // which is exactly the record the reference's in-order loop reports.
  std::vector<ParsedRecord> all(count);
  auto check_range = [&](uint32_t k0, uint32_t k1, int64_t& bad, ParseError& err) {
    for (uint32_t k = k0; k < k1; ++k) {
      try {
        uint64_t off = rd<uint64_t>(data + 10 + 12 * size_t(k));
        uint32_t length = rd<uint32_t>(data + 10 + 12 * size_t(k) + 8);
        std::string ctx = "record " + std::to_string(k);
        if (off + length > len) throw ParseError{RINR_ERR_INTEGRITY, ctx + ": truncated body"};
        if (length < 4) throw ParseError{RINR_ERR_INTEGRITY, ctx + ": record too short for CRC"};
        const uint8_t* blob = data + off;
        uint32_t stored = rd<uint32_t>(blob + length - 4);
        uint32_t actual = crc32(blob, length - 4);
        if (stored != actual) {
          char buf[96];
          std::snprintf(buf, sizeof buf, ": CRC mismatch (stored %#010x, computed %#010x)", stored, actual);
          throw ParseError{RINR_ERR_INTEGRITY, ctx + buf};
        }
        parse_body(blob, length - 4, ctx, all[k]);
        all[k].body_off = off;
      } catch (const ParseError& e) {
        bad = k;
        err = e;
        return;
      }
    }
  };
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const uint32_t nthr = count < 4096 ? 1u : std::min<uint32_t>(std::min(hw, 32u), count / 2048);
  std::vector<int64_t> bad(nthr, -1);
  std::vector<ParseError> errs(nthr);
  if (nthr == 1) {
    check_range(0, count, bad[0], errs[0]);
  } else {
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < nthr; ++t) {
      const uint32_t k0 = uint32_t(uint64_t(count) * t / nthr), k1 = uint32_t(uint64_t(count) * (t + 1) / nthr);
      pool.emplace_back(check_range, k0, k1, std::ref(bad[t]), std::ref(errs[t]));
    }
    for (auto& th : pool) th.join();
  }
  for (uint32_t t = 0; t < nthr; ++t)  // ranges are in index order: the first failing range holds the first failure
    if (bad[t] >= 0) throw errs[t];
  std::vector<std::string> all_ids;
  all_ids.reserve(count);
  for (uint32_t k = 0; k < count; ++k) {
    all_ids.push_back(all[k].id);
    if (keep && k % world == rank) {
      pa.recs.push_back(std::move(all[k]));
      pa.global.push_back(k);
    }
  }
  // ... and finally DatasetArchive's unique-id rule (archive.py:74-77).
  std::unordered_set<std::string> seen;
  seen.reserve(all_ids.size() * 2 + 1);
  for (auto& id : all_ids)
    if (!seen.insert(std::move(id)).second) throw ParseError{RINR_ERR_INVALID_INPUT, "record ids must be unique"};
}

}  // namespace rinr

using namespace rinr;

struct rinr_store {
  int device = 0;
  uint32_t rank = 0, world = 1;
  int64_t total = 0;
  std::vector<HostArch> archs;
  std::vector<int64_t> global;
  std::vector<std::string> ids;
  std::vector<uint32_t> src_h, src_w;
  std::vector<uint16_t> arch_of;
  StoreView view{};
  void* d_alloc = nullptr;  // one device allocation holding every array
  size_t d_bytes = 0;
  int64_t max_record_bytes = 0;
  int64_t max_params = 0;
  bool uniform_arch = true, uniform_source = true;
};

static int cuda_fail(cudaError_t e, const char* what) {
  return set_error(e == cudaErrorMemoryAllocation ? RINR_ERR_OOM : RINR_ERR_CUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

extern "C" {

int rinr_abi_version(void) { return RINR_ABI_VERSION; }

const char* rinr_last_error(void) { return g_err.c_str(); }

int64_t rinr_last_error_record(void) { return g_err_record; }

int rinr_archive_validate(const void* bytes, size_t len, int64_t* count) {
  clear_error();
  if (!bytes && len) return set_error(RINR_ERR_INVALID_INPUT, "null archive buffer");
  try {
    ParsedArchive pa;
    parse_archive(static_cast<const uint8_t*>(bytes), len, 0, 1, pa, false);
    if (count) *count = pa.count;
  } catch (const ParseError& e) {
    int64_t rec = -1;
    if (e.msg.rfind("record ", 0) == 0) rec = std::atoll(e.msg.c_str() + 7);
    return set_error(e.code, e.msg, rec);
  } catch (const std::bad_alloc&) {
    return set_error(RINR_ERR_OOM, "host allocation failed while parsing");
  }
  return RINR_OK;
}

int rinr_archive_shard(const void* bytes, size_t len, uint32_t shard_rank, uint32_t shard_world,
                       int64_t* global_index, int64_t cap, int64_t* count) {
  clear_error();
  if (!bytes && len) return set_error(RINR_ERR_INVALID_INPUT, "null archive buffer");
  if (shard_world < 1 || shard_rank >= shard_world)
    return set_error(RINR_ERR_INVALID_INPUT, "shard_rank must be in [0, shard_world)");
  try {
    ParsedArchive pa;
    parse_archive(static_cast<const uint8_t*>(bytes), len, shard_rank, shard_world, pa, true);
    if (count) *count = int64_t(pa.global.size());
    for (int64_t i = 0; i < int64_t(pa.global.size()) && i < cap && global_index; ++i) global_index[i] = pa.global[i];
  } catch (const ParseError& e) {
    int64_t rec = -1;
    if (e.msg.rfind("record ", 0) == 0) rec = std::atoll(e.msg.c_str() + 7);
    return set_error(e.code, e.msg, rec);
  } catch (const std::bad_alloc&) {
    return set_error(RINR_ERR_OOM, "host allocation failed while parsing");
  }
  return RINR_OK;
}

int rinr_store_create(const void* bytes, size_t len, int device, uint32_t shard_rank, uint32_t shard_world,
                      rinr_store** out) {
  clear_error();
  if (!out) return set_error(RINR_ERR_INVALID_INPUT, "out must not be null");
  *out = nullptr;
  if (shard_world < 1 || shard_rank >= shard_world)
    return set_error(RINR_ERR_INVALID_INPUT, "shard_rank must be in [0, shard_world)");
  std::unique_ptr<rinr_store> st(new rinr_store);
  ParsedArchive pa;
  try {
    parse_archive(static_cast<const uint8_t*>(bytes), len, shard_rank, shard_world, pa, true);
  } catch (const ParseError& e) {
    int64_t rec = -1;
    if (e.msg.rfind("record ", 0) == 0) rec = std::atoll(e.msg.c_str() + 7);
    return set_error(e.code, e.msg, rec);
  } catch (const std::bad_alloc&) {
    return set_error(RINR_ERR_OOM, "host allocation failed while parsing");
  }
  const int64_t n = int64_t(pa.recs.size());
  st->device = device;
  st->rank = shard_rank;
  st->world = shard_world;
  st->total = pa.count;
  st->global = std::move(pa.global);

  // Architecture table + per-record metadata.
  int lmax = 1, maxw = 1;
  st->ids.resize(n);
  st->src_h.resize(n);
  st->src_w.resize(n);
  st->arch_of.resize(n);
  for (int64_t i = 0; i < n; ++i) {
    ParsedRecord& r = pa.recs[i];
    int a = -1;
    for (size_t j = 0; j < st->archs.size(); ++j) {
      const HostArch& h = st->archs[j];
      if (h.nd == r.arch.nd && h.omega == r.arch.omega &&
          std::memcmp(h.dims, r.arch.dims, sizeof(uint16_t) * r.arch.nd) == 0) {
        a = int(j);
        break;
      }
    }
    if (a < 0) {
      if (st->archs.size() >= 65535) return set_error(RINR_ERR_UNSUPPORTED, "more than 65535 architectures");
      st->archs.push_back(r.arch);
      a = int(st->archs.size()) - 1;
    }
    st->arch_of[i] = uint16_t(a);
    lmax = std::max(lmax, r.arch.nd - 1);
    int64_t params = 0;
    for (int l = 0; l + 1 < r.arch.nd; ++l) {
      params += int64_t(r.arch.dims[l]) * r.arch.dims[l + 1] + r.arch.dims[l + 1];
      maxw = std::max(maxw, int(r.arch.dims[l + 1]));
    }
    st->max_params = std::max(st->max_params, params);
    st->max_record_bytes = std::max<int64_t>(st->max_record_bytes, r.body_len);
    st->ids[i] = std::move(r.id);
    st->src_h[i] = r.source_h;
    st->src_w[i] = r.source_w;
    if (i > 0 && (r.source_h != st->src_h[0] || r.source_w != st->src_w[0])) st->uniform_source = false;
  }
  st->uniform_arch = st->archs.size() <= 1;
  bool all_int8 = n > 0;
  for (int64_t i = 0; i < n; ++i) all_int8 = all_int8 && pa.recs[i].hidden_int8;
  const int lstride = lmax + 1;
  const uint32_t hdr = uint32_t((4 * lstride + kRecordAlign - 1) / kRecordAlign * kRecordAlign);
  // Slots: fixed stride when sizes are within 15% of the largest (saves the
  // offset lookup on the kernel's critical path), variable otherwise.
  std::vector<uint64_t> rec_off(n + 1, 0);
  uint64_t sum = 0, max_slot = 0;
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t sl = hdr + (pa.recs[i].body_len + kRecordAlign - 1) / kRecordAlign * kRecordAlign;
    sum += sl;
    max_slot = std::max(max_slot, sl);
  }
  const bool fixed = n > 0 && double(max_slot) * double(n) <= 1.15 * double(sum);
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t sl = fixed ? max_slot : hdr + (pa.recs[i].body_len + kRecordAlign - 1) / kRecordAlign * kRecordAlign;
    rec_off[i + 1] = rec_off[i] + sl;
  }
  const size_t blob = rec_off[n] + kBlobTailPad;

  // Host staging of every device array, then one upload.
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  size_t o_blob = 0, o_rec = al(blob);
  size_t o_aidx = o_rec + al(8 * size_t(n + 1));
  size_t na = std::max<size_t>(st->archs.size(), 1);
  size_t o_adims = o_aidx + al(2 * std::max<int64_t>(n, 1));
  size_t o_and = o_adims + al(2 * na * kMaxDims);
  size_t o_aom = o_and + al(4 * na);
  size_t total = o_aom + al(4 * na);
  std::vector<uint8_t> host;
  try {
    host.assign(total, 0);
  } catch (const std::bad_alloc&) {
    return set_error(RINR_ERR_OOM, "host staging allocation failed");
  }
  const uint8_t* src = static_cast<const uint8_t*>(bytes);
  for (int64_t i = 0; i < n; ++i) {
    const ParsedRecord& r = pa.recs[i];
    uint8_t* slot = host.data() + o_blob + rec_off[i];
    for (size_t l = 0; l < r.lay_off.size(); ++l) std::memcpy(slot + 4 * l, &r.lay_off[l], 4);
    std::memcpy(slot + hdr, src + r.body_off, r.body_len);
  }
  std::memcpy(host.data() + o_rec, rec_off.data(), 8 * size_t(n + 1));
  std::memcpy(host.data() + o_aidx, st->arch_of.data(), 2 * n);
  for (size_t a = 0; a < st->archs.size(); ++a) {
    const HostArch& h = st->archs[a];
    std::memcpy(host.data() + o_adims + 2 * a * kMaxDims, h.dims, 2 * h.nd);
    int32_t nd = h.nd;
    std::memcpy(host.data() + o_and + 4 * a, &nd, 4);
    float om = float(h.omega);
    std::memcpy(host.data() + o_aom + 4 * a, &om, 4);
  }
  pa.recs.clear();

  int prev = 0;
  cudaError_t e = cudaGetDevice(&prev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  e = cudaMalloc(&st->d_alloc, total);
  if (e == cudaSuccess) e = cudaMemcpy(st->d_alloc, host.data(), total, cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    if (st->d_alloc) cudaFree(st->d_alloc);
    st->d_alloc = nullptr;
    return cuda_fail(e, "store upload");
  }
  st->d_bytes = total;
  uint8_t* d = static_cast<uint8_t*>(st->d_alloc);
  StoreView& v = st->view;
  v.blob = d + o_blob;
  v.rec_off = reinterpret_cast<const uint64_t*>(d + o_rec);
  v.arch_idx = reinterpret_cast<const uint16_t*>(d + o_aidx);
  v.arch_dims = reinterpret_cast<const uint16_t*>(d + o_adims);
  v.arch_nd = reinterpret_cast<const int32_t*>(d + o_and);
  v.arch_omega = reinterpret_cast<const float*>(d + o_aom);
  v.n = n;
  v.lstride = lstride;
  v.hdr_bytes = int32_t(hdr);
  v.slot_stride = fixed ? int64_t(max_slot) : 0;
  v.n_arch = int32_t(st->archs.size());
  v.max_slot_bytes = int32_t(max_slot);
  v.max_params = int32_t(st->max_params);
  v.max_width = maxw;
  v.hidden_int8 = all_int8 ? 1 : 0;
  *out = st.release();
  return RINR_OK;
}

int rinr_store_destroy(rinr_store* store) {
  clear_error();
  if (!store) return RINR_OK;
  if (store->d_alloc) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(store->device);
    cudaError_t e = cudaFree(store->d_alloc);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      delete store;
      return cuda_fail(e, "cudaFree");
    }
  }
  delete store;
  return RINR_OK;
}

int rinr_store_info(const rinr_store* s, rinr_store_info_t* info) {
  clear_error();
  if (!s || !info) return set_error(RINR_ERR_INVALID_INPUT, "null store or info");
  std::memset(info, 0, sizeof *info);
  info->num_records = s->view.n;
  info->total_records = s->total;
  info->shard_rank = s->rank;
  info->shard_world = s->world;
  info->device = s->device;
  info->uniform_arch = s->uniform_arch ? 1 : 0;
  if (!s->archs.empty()) {
    info->n_dims = s->archs[0].nd;
    std::memcpy(info->dims, s->archs[0].dims, 2 * s->archs[0].nd);
    info->omega = s->archs[0].omega;
  }
  info->max_param_count = s->max_params;
  info->max_record_bytes = s->max_record_bytes;
  info->device_bytes = int64_t(s->d_bytes);
  info->uniform_source = s->uniform_source ? 1 : 0;
  if (!s->src_h.empty()) {
    info->source_h = s->src_h[0];
    info->source_w = s->src_w[0];
  }
  return RINR_OK;
}

int rinr_store_record_meta(const rinr_store* s, int64_t k, int64_t* global_index, char* id_buf, size_t id_cap,
                           size_t* id_len, uint32_t* source_h, uint32_t* source_w) {
  clear_error();
  if (!s) return set_error(RINR_ERR_INVALID_INPUT, "null store");
  if (k < 0 || k >= s->view.n)
    return set_error(RINR_ERR_INVALID_INPUT,
                     "record " + std::to_string(k) + " out of range [0, " + std::to_string(s->view.n) + ")");
  if (global_index) *global_index = s->global[k];
  const std::string& id = s->ids[k];
  if (id_len) *id_len = id.size();
  if (id_buf && id_cap) {
    size_t m = std::min(id_cap - 1, id.size());
    std::memcpy(id_buf, id.data(), m);
    id_buf[m] = 0;
  }
  if (source_h) *source_h = s->src_h[k];
  if (source_w) *source_w = s->src_w[k];
  return RINR_OK;
}

}  // extern "C"

namespace {
// Launch on the store's device whatever the caller's current device is; a
// no-op (one cudaGetDevice) when they already match, so it is capture-safe.
struct StoreDevice {
  int prev = -1;
  explicit StoreDevice(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~StoreDevice() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

int rinr_dequantize(const rinr_store* s, const int64_t* d_ids, int64_t n, float* d_out, int64_t out_stride,
                    int32_t* d_status, void* stream) {
  clear_error();
  if (!s) return set_error(RINR_ERR_INVALID_INPUT, "null store");
  if (n < 0) return set_error(RINR_ERR_INVALID_INPUT, "n must be >= 0");
  if (n == 0) return RINR_OK;
  if (!d_ids || !d_out) return set_error(RINR_ERR_INVALID_INPUT, "null ids or output");
  if (out_stride < s->max_params)
    return set_error(RINR_ERR_INVALID_INPUT, "out_stride " + std::to_string(out_stride) +
                                                 " < max_param_count " + std::to_string(s->max_params));
  StoreDevice guard(s->device);
  return rinr_launch_dequantize(s->view, d_ids, n, d_out, out_stride, d_status, stream);
}

int rinr_decode(const rinr_store* s, const int64_t* d_ids, int64_t n, const rinr_decode_params_t* p,
                const float* d_aug, void* d_out, int32_t* d_status, void* stream) {
  clear_error();
  if (!s || !p) return set_error(RINR_ERR_INVALID_INPUT, "null store or params");
  if (p->out_h < 1 || p->out_w < 1)
    return set_error(RINR_ERR_INVALID_INPUT,
                     "output size must be >= 1x1, got " + std::to_string(p->out_h) + "x" + std::to_string(p->out_w));
  if (n < 0) return set_error(RINR_ERR_INVALID_INPUT, "n must be >= 0");
  if (n == 0) return RINR_OK;
  if (!d_ids || !d_out) return set_error(RINR_ERR_INVALID_INPUT, "null ids or output");
  if (p->out_dtype < 0 || p->out_dtype > RINR_OUT_U8 || p->out_layout < 0 || p->out_layout > RINR_LAYOUT_NHWC ||
      p->precision < 0 || p->precision > RINR_PREC_EXACT || p->sin_mode < 0 || p->sin_mode > RINR_SIN_ACCURATE ||
      p->aug_mode < 0 || p->aug_mode > RINR_AUG_CROP)
    return set_error(RINR_ERR_INVALID_INPUT, "decode parameter out of range");
  if ((p->aug_mode != RINR_AUG_NONE) != (d_aug != nullptr))
    return set_error(RINR_ERR_INVALID_INPUT, "d_aug must be given iff aug_mode != NONE");
  for (int c = 0; c < 3; ++c)
    if (!(p->std[c] != 0.0f)) return set_error(RINR_ERR_INVALID_INPUT, "std must be non-zero");
  if (int64_t(p->out_h) * p->out_w > (int64_t(1) << 31) / 4)
    return set_error(RINR_ERR_INVALID_INPUT, "output image too large");
  const HostArch* ua = (s->uniform_arch && !s->archs.empty()) ? &s->archs[0] : nullptr;
  StoreDevice guard(s->device);
  return rinr_launch_decode(s->view, ua, d_ids, n, p, d_aug, d_out, d_status, stream);
}

}  // extern "C"
