// Microbenchmark (development only): T warps each issue a chain of `len`
// tcgen05.mma (M128 N48 K16, A in TMEM) into their own accumulator and commit
// to their own mbarrier, concurrently ("free"), or one chain at a time under a
// shared-memory lock ("lock"), or all chains issued by warp 0 ("one").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2306_16699_b200/csrc tools/micro/umma_multi.cu -o tools/micro/umma_multi
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_decode.cuh"

using namespace rinr;

__global__ void __launch_bounds__(256, 1) umma_multi(int T, int len, int mode, int rounds, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[8];
  __shared__ uint32_t tslot;
  __shared__ int lock;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 24 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (tid < 8) tc::mbar_init(&mbar[tid], 1);
  if (tid == 0) lock = 0;
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
  long long tot = 0;
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    auto chain = [&](int c) {
      const uint32_t d = tmem + uint32_t(c * 96), a = d + 48;
      for (int k = 0; k < len; ++k) {
        const int ks = k % 3;
        tc::mma_bf16_ts_warp(d, a + uint32_t(ks * 8), tc::make_desc(bsm + ks * 256, 128, 6 * 128), idesc, k > 0);
      }
      tc::commit_warp(&mbar[c]);
    };
    if (mode == 2) {
      if (warp == 0)
        for (int c = 0; c < T; ++c) chain(c);
    } else if (warp < T) {
      if (mode == 1) {
        if (tid % 32 == 0) while (atomicCAS(&lock, 0, 1) != 0) {}
        __syncwarp();
        chain(warp);
        __syncwarp();
        if (tid % 32 == 0) atomicExch(&lock, 0);
      } else {
        chain(warp);
      }
    }
    if (warp < T) tc::mbar_wait(&mbar[warp], phase);
    phase ^= 1u;
    tc::fence_after();
    __syncthreads();
    const long long t1 = clock64();
    if (r > 0) tot += t1 - t0;
  }
  if (tid == 0) out[0] = tot / (rounds - 1);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(umma_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * 1024);
  const char* names[3] = {"free", "lock", "one "};
  for (int len : {3, 6})
    for (int T : {1, 2, 5})
      for (int mode = 0; mode < 3; ++mode) {
        umma_multi<<<1, 256, 24 * 1024>>>(T, len, mode, 50, d);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("error\n"); return 1; }
        long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("len %d T %d %s: %6lld cycles per round, %6.1f per MMA\n", len, T, names[mode], h, double(h) / (T * len));
      }
  return 0;
}
