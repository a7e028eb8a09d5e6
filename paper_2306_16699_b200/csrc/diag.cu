// Pipe-peak microbenchmarks used as roofline denominators by bench.py.
// MEASURED_PEAKS.json holds only HBM copy and cuBLAS bf16 rates; the decode is
// bound by the SFU (MUFU) pipe, so its peak is measured here on the same GPU
// and in the same run as the decode it normalises.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/rinr_b200_diag.h"

namespace {

// 8 independent chains per thread; every iteration issues 8 MUFU.SIN.
__global__ void diag_mufu(int iters, float* sink) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = float(threadIdx.x) * 1e-3f + float(j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __sinf(x[j]);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) sink[0] = s;
}

// 8 independent FFMA chains per thread (2 flops each).
__global__ void diag_ffma(int iters, float* sink) {
  float x[8];
  const float a = 0.999f, b = 1e-4f;
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = float(threadIdx.x) + float(j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) sink[0] = s;
}

// 4 independent mma.sync.m16n8k16 bf16 accumulator chains per warp.
__global__ void diag_hmma(int iters, float* sink) {
  uint32_t a[4] = {0x3f803f80u ^ threadIdx.x, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u};
  uint32_t b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  float d[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};\n"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1234.5f) sink[0] = s;
}

}  // namespace

extern "C" RINR_API int rinr_diag_launch(int kind, int blocks, int threads, int iters, float* d_sink, void* stream,
                                         double* ops_per_launch) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double ops = 0.0;
  switch (kind) {
    case RINR_DIAG_MUFU_SIN:
      diag_mufu<<<blocks, threads, 0, st>>>(iters, d_sink);
      ops = double(blocks) * threads * iters * 8.0;  // sines
      break;
    case RINR_DIAG_FFMA:
      diag_ffma<<<blocks, threads, 0, st>>>(iters, d_sink);
      ops = double(blocks) * threads * iters * 8.0 * 2.0;  // flops
      break;
    case RINR_DIAG_HMMA_BF16:
      diag_hmma<<<blocks, threads, 0, st>>>(iters, d_sink);
      ops = double(blocks) * (threads / 32) * iters * 4.0 * (2.0 * 16 * 8 * 16);  // flops
      break;
    default:
      return RINR_ERR_INVALID_INPUT;
  }
  if (ops_per_launch) *ops_per_launch = ops;
  return cudaPeekAtLastError() == cudaSuccess ? RINR_OK : RINR_ERR_CUDA;
}
