// mmaprobe.cu — tcgen05.mma (TS, M=128, fp16 -> fp32) issue cost and
// issue->commit->mbarrier round trip, unrolled with warp-uniform operands.
//   case 0: fence + commit only
//   case k (1..8): k MMAs into ONE accumulator (dependent) + commit
//   case 10+k: k MMAs into k DIFFERENT accumulators (independent) + commit
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace nmq;
template <int N, int K, bool INDEP>
__global__ void rt_bench(int reps, long long* out) {
  __shared__ __align__(1024) uint8_t sB[16384];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (tid < 32) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async_smem(); tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
  constexpr uint32_t idesc = tc::idesc_f16(128, N);
  const uint64_t bd = tc::smem_desc(tc::smem_u32(sB), N * 16, 128);
  long long issue = 0, total = 0;
  if (tid < 32) {
    for (int rep = 0; rep < reps; ++rep) {
      __syncwarp();
      long long t0 = clock64(), t1 = 0;
      if (tid == 0) {
        tc::tc_fence_after();
#pragma unroll
        for (int i = 0; i < K; ++i)
          tc::mma_ts(INDEP ? tb + 32 * i : tb, tb + 384 + 8 * (i & 7), bd + ((i * 2 * N * 16) >> 4), idesc,
                     INDEP ? 0 : (i > 0));
        tc::mma_commit(&bar);
        t1 = clock64();
      }
      __syncwarp();
      tc::mbar_wait(&bar, rep & 1);
      tc::tc_fence_after();
      long long t2 = clock64();
      if (rep > 0) { issue += t1 - t0; total += t2 - t0; }
    }
    if (tid == 0) { out[0] = issue / (reps - 1); out[1] = total / (reps - 1); }
  }
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  if (tid < 32) tc::tmem_free<512>(tb);
}
template <int N, int K, bool INDEP>
void run() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  rt_bench<N, K, INDEP><<<1, 128>>>(50, d); cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("N=%3d k=%d %s: issue %5lld cyc, issue->complete %5lld cyc\n", N, K, INDEP ? "indep" : "chain", h[0], h[1]);
  cudaFree(d);
}
int main() {
  run<32, 0, false>();
  run<16, 1, false>(); run<32, 1, false>();
  run<32, 2, false>(); run<32, 3, false>(); run<32, 5, false>(); run<32, 8, false>();
  run<32, 2, true>(); run<32, 5, true>(); run<32, 8, true>();
  run<64, 5, false>(); run<128, 5, false>(); run<256, 5, false>();
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
