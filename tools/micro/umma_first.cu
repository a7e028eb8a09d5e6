// Microbenchmark (development only): where does the ~400-cycle issue latency
// of the first tcgen05.mma of a sequence come from?  One warp, elect-issued.
//   mode 0: [mma x len, commit], wait, fence_after         (baseline)
//   mode 1: same without tcgen05.fence::after_thread_sync
//   mode 2: two sequences per round on the same D, commit between, one wait
//   mode 3: two sequences per round on different D, commit between, one wait
//   mode 4: baseline preceded by a tcgen05.st + wait::st by the whole warp
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2306_16699_b200/csrc tools/micro/umma_first.cu -o tools/micro/umma_first
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_decode.cuh"

using namespace rinr;

__global__ void __launch_bounds__(128, 1) umma_first(int len, int mode, int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 24 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (tid < 2) tc::mbar_init(&mbar[tid], 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  const uint32_t idesc = tc::make_idesc(128, 48);
  const uint32_t bsm = tc::smem_u32(smem);
  uint32_t phase = 0;
  long long t_first = 0, t_all = 0;
  if (warp == 0) {
    for (int r = 0; r < rounds; ++r) {
      if (mode == 4) {
        uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        tc::tmem_st8(tmem + 48, z);
        tc::tmem_wait_st();
        tc::fence_before();
        __syncwarp();
        tc::fence_after();
      }
      const long long t0 = clock64();
      long long t1 = 0;
      const int seqs = (mode == 2 || mode == 3) ? 2 : 1;
      for (int q = 0; q < seqs; ++q) {
        const uint32_t d = tmem + uint32_t(mode == 3 ? q * 128 : 0), a = tmem + 48;
        for (int k = 0; k < len; ++k) {
          const int ks = k % 3;
          tc::mma_bf16_ts_warp(d, a + uint32_t(ks * 8), tc::make_desc(bsm + ks * 256, 128, 6 * 128), idesc, k > 0);
          if (q == 0 && k == 0) t1 = clock64();
        }
        tc::commit_warp(&mbar[0]);
        if (q + 1 < seqs) {  // wait for the first sequence before the second (phase flips)
          tc::mbar_wait(&mbar[0], phase);
          phase ^= 1u;
        }
      }
      tc::mbar_wait(&mbar[0], phase);
      phase ^= 1u;
      if (mode != 1) tc::fence_after();
      const long long t2 = clock64();
      if (r > 0) {
        t_first += t1 - t0;
        t_all += t2 - t0;
      }
    }
    if (tid == 0) {
      out[0] = t_first / (rounds - 1);
      out[1] = t_all / (rounds - 1);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(umma_first, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024);
  for (int mode = 0; mode < 5; ++mode)
    for (int len : {1, 3, 6}) {
      umma_first<<<1, 128, 24 * 1024>>>(len, mode, 50, d);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("mode %d len %d: first-MMA issue %5lld cycles, round %5lld cycles\n", mode, len, h[0], h[1]);
    }
  return 0;
}
