/*
 * rinr_b200.h — C ABI of the B200-native Rapid-INR batched decode.
 *
 * The reference (Rapid-INR, arXiv 2306.16699; /root/reference/pkg/src/rinr)
 * exposes its decode path as module-level Python functions, not an FFI.  Each
 * entry point below replaces one of them; the reference interface it stands in
 * for is cited next to it.  Plain C types only: device pointers are `void*` /
 * typed pointers allocated by the caller (e.g. torch tensors), streams are
 * `cudaStream_t` passed as `void*`.  Every call returns a status code
 * (RINR_OK or one of the error codes below) and leaves a thread-local message
 * readable through rinr_last_error().
 *
 * Error codes map 1:1 onto the reference's exception taxonomy
 * (errors.py:8-50): RINR_ERR_INVALID_INPUT -> InvalidInputError,
 * RINR_ERR_FORMAT -> FormatError, RINR_ERR_INTEGRITY -> IntegrityError
 * (the failing record index is reported), RINR_ERR_CUDA / RINR_ERR_OOM ->
 * RuntimeError / MemoryError on the Python side.
 */
#ifndef RINR_B200_H
#define RINR_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RINR_API __attribute__((visibility("default")))
#else
#define RINR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define RINR_ABI_VERSION 1

enum rinr_status {
  RINR_OK = 0,
  RINR_ERR_INVALID_INPUT = 1, /* InvalidInputError (errors.py:12)          */
  RINR_ERR_FORMAT = 2,        /* FormatError       (errors.py:32)          */
  RINR_ERR_INTEGRITY = 3,     /* IntegrityError    (errors.py:36-41)       */
  RINR_ERR_CUDA = 4,          /* CUDA runtime failure                      */
  RINR_ERR_OOM = 5,           /* device or host allocation failed          */
  RINR_ERR_UNSUPPORTED = 6,   /* valid record this build cannot decode     */
  RINR_ERR_STRUCTURAL = 7,    /* StructuralError   (errors.py:28)          */
  RINR_ERR_NUMERIC = 8        /* NumericError      (errors.py:16)          */
};

/* Output element type / layout of rinr_decode. */
enum rinr_out_dtype { RINR_OUT_F32 = 0, RINR_OUT_BF16 = 1, RINR_OUT_U8 = 2 };
enum rinr_out_layout { RINR_LAYOUT_NCHW = 0, RINR_LAYOUT_NHWC = 1 };

/* Arithmetic of the hidden-layer contractions.
 *   RINR_PREC_FP32 : bf16x3 split on tensor cores (hi*hi + hi*lo + lo*hi),
 *                    fp32 accumulate; max-abs <= 1e-3 vs the CPU oracle.
 *   RINR_PREC_BF16 : one bf16 pass, fp32 accumulate; stated as a PSNR delta.
 *   RINR_PREC_EXACT: plain fp32 FFMA on CUDA cores, any architecture (the
 *                    correctness anchor; also used for non-uniform archs). */
enum rinr_precision { RINR_PREC_FP32 = 0, RINR_PREC_BF16 = 1, RINR_PREC_EXACT = 2 };

/* Sine evaluation: MUFU (__sinf) or the accurate libdevice sinf. */
enum rinr_sin_mode { RINR_SIN_MUFU = 0, RINR_SIN_ACCURATE = 1 };

/* Coordinate transform applied before the MLP (crop / flip; not in the
 * reference — SPEC.md:8 puts augmentation out of scope — so this repo defines
 * it; oracle/rinr_oracle.py:augment_coords is the checker).
 *   RINR_AUG_NONE  : the reference coordinate grid (net.py:138-149).
 *   RINR_AUG_OFFSET: per image {dx, dy, flip, pad, 0}: integer pixel offset
 *                    crop with zero padding (CIFAR pad-4 random crop).
 *   RINR_AUG_CROP  : per image {x0, y0, sx, sy, flip}: continuous crop box in
 *                    normalised source coordinates (random-resized crop). */
enum rinr_aug_mode { RINR_AUG_NONE = 0, RINR_AUG_OFFSET = 1, RINR_AUG_CROP = 2 };

typedef struct rinr_store rinr_store;

typedef struct {
  int64_t num_records;     /* records resident in this shard                 */
  int64_t total_records;   /* records in the archive                          */
  uint32_t shard_rank;
  uint32_t shard_world;
  int32_t device;
  int32_t uniform_arch;    /* 1: every record has the same dims and omega    */
  int32_t n_dims;          /* dims of record 0 (of every record if uniform)  */
  uint16_t dims[32];
  double omega;
  int64_t max_param_count; /* floats per record written by rinr_dequantize   */
  int64_t max_record_bytes;
  int64_t device_bytes;    /* HBM held by the store                          */
  int32_t uniform_source;  /* 1: every record has the same source_h/w        */
  uint32_t source_h;
  uint32_t source_w;
} rinr_store_info_t;

typedef struct {
  int32_t out_h, out_w;    /* >= 1; decode resolution (decoder.py:26-29)     */
  int32_t out_dtype;       /* rinr_out_dtype                                 */
  int32_t out_layout;      /* rinr_out_layout                                */
  int32_t precision;       /* rinr_precision                                 */
  int32_t sin_mode;        /* rinr_sin_mode                                  */
  int32_t aug_mode;        /* rinr_aug_mode                                  */
  float mean[3];           /* epilogue: (clamp(v) - mean) / std per channel  */
  float std[3];
  int32_t flags;           /* RINR_FLAG_* bits                               */
} rinr_decode_params_t;

/* flags: the ids / aug inputs were not written by the kernel that precedes this
 * decode on the stream (e.g. they came from a host copy, or the previous launch
 * is another decode), so the prologue (record fetch + dequantisation) may start
 * while that kernel drains (programmatic dependent launch); outputs are still
 * written only after it completes. */
#define RINR_FLAG_OVERLAP_PROLOGUE 1
/* flags: `ids` holds 2n entries, this batch then the next one (training
 * samplers know it); the narrow-net kernel prefetches the next batch's record
 * slots into L2 while it decodes this one.  Output covers the first n only. */
#define RINR_FLAG_PREFETCH_NEXT 2

/* Version of this ABI (RINR_ABI_VERSION). */
RINR_API int rinr_abi_version(void);

/* Thread-local message of the last failing call on this thread ("" if none). */
RINR_API const char* rinr_last_error(void);
/* Record index named by the last RINR_ERR_INTEGRITY / per-item error, or -1
 * (IntegrityError.record / BatchItemError.index). */
RINR_API int64_t rinr_last_error_record(void);

/* Host-only validation of a whole .rinr image (no GPU needed): header, chained
 * index, per-record CRC32, record parse and unique ids — the checks
 * rinr.read() performs (archive.py:338-400).  Replaces ArchiveReader(...) +
 * read_raw(k) for every k.  On success *count = number of records. */
RINR_API int rinr_archive_validate(const void* bytes, size_t len, int64_t* count);

/* Host-only: global indices of the records rinr_store_create(..., shard_rank,
 * shard_world, ...) keeps (k % shard_world == shard_rank), after the same full
 * validation.  Writes up to `cap` indices; *count = shard size. */
RINR_API int rinr_archive_shard(const void* bytes, size_t len, uint32_t shard_rank, uint32_t shard_world,
                                int64_t* global_index, int64_t cap, int64_t* count);

/* Parse + validate an archive image held in host memory and upload the
 * records whose index k satisfies k % shard_world == shard_rank to `device`
 * HBM.  Replaces rinr.read(source) (archive.py:395-400) + the materialise step
 * (archive.py:278-325), which now happens inside every decode.  The store is
 * immutable; concurrent decodes on different streams are safe. */
RINR_API int rinr_store_create(const void* bytes, size_t len, int device,
                      uint32_t shard_rank, uint32_t shard_world, rinr_store** out);
RINR_API int rinr_store_destroy(rinr_store* store);
RINR_API int rinr_store_info(const rinr_store* store, rinr_store_info_t* info);

/* Metadata of one resident record by local index (archive.py:61-65,
 * ArchiveRecord.id / InrModel.source_h/w).  `id_buf` receives the UTF-8 id,
 * NUL-terminated and truncated to id_cap; *id_len gets its full length. */
RINR_API int rinr_store_record_meta(const rinr_store* store, int64_t local_index, int64_t* global_index,
                           char* id_buf, size_t id_cap, size_t* id_len, uint32_t* source_h,
                           uint32_t* source_w);

/* Bit-exact integer dequantisation hook: for each of the n local record ids in
 * d_ids (device int64), write the materialised parameters
 * [w0 (out x in, row-major), b0, w1, b1, ...] as f32 into
 * d_out + i * out_stride (floats).  Exactly archive.materialize
 * (archive.py:278-325): affine codes -> f32(f64 scale * (f64 code - zp)),
 * masked entries +0.0, f32/f16 layers scattered/copied (f16 widened exactly).
 * Stream-ordered, no host sync.  d_status as in rinr_decode. */
RINR_API int rinr_dequantize(const rinr_store* store, const int64_t* d_ids, int64_t n, float* d_out,
                    int64_t out_stride, int32_t* d_status, void* stream);

/* Fused batched decode: for each of the n local record ids in d_ids, dequantise
 * the record in the kernel prologue, evaluate its SIREN MLP at every output
 * coordinate (after the optional crop/flip transform), clamp to [0,1],
 * normalise and store image i at d_out + i * (3*out_h*out_w) elements in the
 * requested dtype/layout.  Replaces decoder.decode_batch (decoder.py:39-61)
 * / decode (decoder.py:19-36) and the CPU augmentation a data loader would run.
 * d_aug: device float[n*5] per-image parameters (NULL iff aug_mode == NONE).
 * d_status: optional device int32; reset by this call, after the stream
 * reaches it holds 0, or (n - i) for the first id i that is out of range
 * (-> BatchItemError(i, InvalidInputError)).  Stream-ordered, no host sync.
 * Both calls launch on the store's device (rinr_store_create's `device`)
 * whatever the caller's current device is; `stream` and every pointer must
 * belong to that device. */
RINR_API int rinr_decode(const rinr_store* store, const int64_t* d_ids, int64_t n,
                const rinr_decode_params_t* params, const float* d_aug, void* d_out,
                int32_t* d_status, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RINR_B200_H */
