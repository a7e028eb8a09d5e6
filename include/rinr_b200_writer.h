/* GPU .rinr writer: serialise a device-resident batch of same-architecture
 * models into archive bytes in device memory (the
 * GPU-side synthetic store generator).  Replaces the reference writer
 * archive.serialize / archive.write (archive.py:161-184) and its per-record
 * encoder (encode_record, _encode_layer, _layer_plan: archive.py:92-158) for
 * batches produced on the GPU by rinr_prune_l1 / rinr_quantize; the bytes are
 * identical to the reference writer's (tests/test_gpu_writer.py).
 *
 * Inputs use the transform layout of rinr_b200_transforms.h:
 *   d_w     [n][P] f32, d_mask [n][P] u8, d_b [n][sum dims[1..]] f32;
 *   quant_bits 0 (no quantisation: every layer f32) or 8 / 16, then
 *   d_scale / d_zp / d_const [n][nl-2] and d_codes [n][P] u16 as written by
 *   rinr_quantize (hidden layers 1..nl-2).
 * Record k's id is id_prefix followed by first_id + k in decimal, zero padded
 * to id_width digits (Python f"{prefix}{first_id + k:0{id_width}d}").
 *
 * Two calls: rinr_serialize_size writes every record's length (CRC
 * included) plus per-layer forms / kept counts; the caller scans the lengths
 * into byte offsets (exclusive prefix sum, relative to the first record) and
 * allocates 10 + 12 n + sum(lengths) bytes; rinr_serialize_write fills the
 * header, the index and every record (CRC-32 last).  Both are asynchronous on
 * `stream`. */
#ifndef RINR_B200_WRITER_H
#define RINR_B200_WRITER_H

#include <stddef.h>
#include <stdint.h>

#include "rinr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  const int32_t* dims; /* host: n_layers + 1 widths, 2 ... 3 */
  int n_layers;
  int64_t n;
  uint32_t source_h, source_w;
  double omega;
  int quant_bits;
  const float* d_w;
  const uint8_t* d_mask;
  const float* d_b;
  const double* d_scale;
  const int32_t* d_zp;
  const uint8_t* d_const;
  const uint16_t* d_codes;
  const char* id_prefix; /* host, < 48 bytes, may be NULL */
  int64_t first_id;
  int id_width;
} rinr_serialize_args_t;

/* d_rec_len [n] i64, d_forms [n][n_layers] u8, d_kept [n][n_layers] i32. */
RINR_API int rinr_serialize_size(const rinr_serialize_args_t* args, int64_t* d_rec_len, uint8_t* d_forms,
                                 int32_t* d_kept, void* stream);

/* d_rec_off [n] i64: exclusive prefix sum of d_rec_len; d_out: the archive. */
RINR_API int rinr_serialize_write(const rinr_serialize_args_t* args, const int64_t* d_rec_off, const int64_t* d_rec_len,
                                  const uint8_t* d_forms, const int32_t* d_kept, uint8_t* d_out, void* stream);

#ifdef __cplusplus
}
#endif

#endif
