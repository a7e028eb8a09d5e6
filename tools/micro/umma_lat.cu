// Microbenchmark (development only, not part of the library): latency and
// throughput of chains of tcgen05.mma kind::f16 M=128 x N x K=16 with A in
// TMEM (.ts) or shared memory (.ss), B in shared memory, issued by one thread
// into `chains` independent accumulators of `len` MMAs each, one commit per
// chain.  Prints cycles per round (issue and completion) for each shape.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -I paper_2306_16699_b200/csrc tools/micro/umma_lat.cu -o tools/micro/umma_lat
#include <cstdio>
#include <cuda_runtime.h>
#include "tc_decode.cuh"

using namespace rinr;

// whole-warp issue: every lane computes the (uniform) operands, elect.sync
// picks the issuing lane inside the asm
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\t"
      "elect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(tc::smem_u32(mbar))
      : "memory");
}

template <int N, bool SS, bool WARP = false>
__global__ void __launch_bounds__(128, 1) umma_chain(int chains, int len, int rounds, long long* out, int one_commit, int acc_always) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar[8];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (tid < 8) tc::mbar_init(&mbar[tid], 1);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tslot;
  constexpr uint32_t K = 48, CH = K / 8;
  const uint32_t idesc = tc::make_idesc(128, N);
  const uint32_t bsm = tc::smem_u32(smem);            // B: N x 48 bf16 K-major
  const uint32_t asm_ = tc::smem_u32(smem + 24576);   // A (SS): 128 x 48 bf16 K-major
  const int dcols = N;                                // f32 accumulator columns
  const int stride = 512 / 8;                         // columns per chain region (8 chains max)
  uint32_t phase = 0;
  long long t_iss = 0, t_all = 0;
  if (WARP ? tid < 32 : tid == 0) {
    for (int r = 0; r < rounds; ++r) {
      const long long t0 = clock64();
      for (int c = 0; c < chains; ++c) {
        const uint32_t d = tmem + uint32_t(c * (N <= 32 ? stride : 96 * 0 + (512 / chains) / 16 * 16));
        const uint32_t a = d + uint32_t(dcols);
        for (int k = 0; k < len; ++k) {
          const int ks = k % 3;
          const uint64_t bdesc = tc::make_desc(bsm + ks * 256, 128, CH * 128);
          if constexpr (WARP) {
            mma_ts_elect(d, a + uint32_t(ks * 8), bdesc, idesc, acc_always || k > 0);
          } else if constexpr (SS) {
            const uint64_t adesc = tc::make_desc(asm_ + ks * 256, 128, CH * 128);
            tc::mma_bf16(d, adesc, bdesc, idesc, k > 0);
          } else {
            tc::mma_bf16_ts(d, a + uint32_t(ks * 8), bdesc, idesc, acc_always || k > 0);
          }
        }
        if (!one_commit || c == chains - 1) {
          if constexpr (WARP) commit_elect(&mbar[c]);
          else tc::commit(&mbar[c]);
        }
      }
      const long long t1 = clock64();
      for (int c = one_commit ? chains - 1 : 0; c < chains; ++c) tc::mbar_wait(&mbar[c], phase);
      phase ^= 1u;
      tc::fence_after();
      const long long t2 = clock64();
      if (r > 0) {
        t_iss += t1 - t0;
        t_all += t2 - t0;
      }
    }
    if (tid == 0) {
      out[blockIdx.x * 2 + 0] = t_iss / (rounds - 1);
      out[blockIdx.x * 2 + 1] = t_all / (rounds - 1);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int N, bool SS, bool WARP = false>
void run(int chains, int len, int grid, int one_commit = 0, int acc_always = 0) {
  long long* d;
  cudaMalloc(&d, 2 * 1024 * sizeof(long long));
  auto k = umma_chain<N, SS, WARP>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  k<<<grid, 128, 48 * 1024>>>(chains, len, 50, d, one_commit, acc_always);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  const double per = double(h[1]) / (chains * len);
  printf("%s%s%s N=%3d %s chains=%d len=%2d grid=%3d: issue %6lld cyc, done %6lld cyc per round -> %6.1f cyc/MMA, %6.0f MAC/clk\n",
         acc_always ? "acc1 " : "     ", one_commit ? "1c " : "   ", WARP ? "warp" : "thr ", N, SS ? "ss" : "ts", chains, len, grid, h[0], h[1], per, 128.0 * N * 16 / per);
  cudaFree(d);
}

int main() {
  for (int g : {1}) {
    run<48, false, true>(5, 6, g, 0, 1);
    run<48, false, true>(1, 6, g, 0, 1);
    run<48, false, true>(1, 1, g, 0, 1);
    run<48, false, false>(5, 6, g, 0, 1);
    run<48, false, true>(5, 6, g, 1);
    run<48, false, true>(5, 3, g, 1);
    run<48, false, false>(5, 6, g, 1);
    run<48, false, true>(1, 30, g, 1);
    run<48, false, true>(1, 1, g);
    run<48, false, true>(1, 6, g);
    run<48, false, true>(1, 12, g);
    run<48, false, true>(5, 6, g);
    run<48, false, true>(5, 3, g);
    run<48, false>(1, 1, g);
    run<48, false>(1, 6, g);
    run<48, false>(1, 12, g);
    run<48, false>(2, 6, g);
    run<48, false>(5, 6, g);
    run<48, true>(1, 6, g);
    run<48, true>(5, 6, g);
    run<64, false>(1, 6, g);
    run<64, false>(5, 6, g);
    run<128, false>(1, 6, g);
    run<128, false>(3, 6, g);
    run<256, false>(1, 6, g);
    run<16, false>(1, 6, g);
    run<16, false>(5, 6, g);
  }
  return 0;
}
