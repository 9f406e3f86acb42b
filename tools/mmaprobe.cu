// mmaprobe.cu — issue cost of tcgen05.mma (TS, M=128, N=32, K=16): dependent
// chain on one accumulator vs alternating independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"
using namespace nmq;
__global__ void issue_bench(int iters, int mode, long long* out) {
  __shared__ __align__(1024) uint8_t sB[8192];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < 2048; i += blockDim.x) reinterpret_cast<uint32_t*>(sB)[i] = 0;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (tid < 32) tc::tmem_alloc<512>(&tbase);
  tc::fence_proxy_async_smem(); tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tbase, 0);
  const uint32_t idesc = tc::idesc_f16(128, 32);
  const uint64_t bd = tc::smem_desc(tc::smem_u32(sB), 32 * 16, 128);
  long long t0 = 0, t1 = 0, t2 = 0;
  if (tid < 32) {
    for (int rep = 0; rep < 2; ++rep) {
      if (tid == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
          uint32_t d = (mode == 0) ? tb : tb + 32 * (i & 7);
          tc::mma_ts(d, tb + 256 + 8 * (i & 3), bd, idesc, 1);
        }
        t1 = clock64();
        tc::mma_commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, rep & 1);
      t2 = clock64();
    }
    if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  tc::tc_fence_before(); __syncthreads(); tc::tc_fence_after();
  if (tid < 32) tc::tmem_free<512>(tb);
}
int main() {
  long long* d; cudaMalloc(&d, 16); long long h[2];
  for (int mode = 0; mode < 2; ++mode)
    for (int iters : {1, 4, 16, 64}) {
      issue_bench<<<1, 128>>>(iters, mode, d); cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("mode=%s iters=%d: issue %lld cyc (%.1f/mma), complete %lld cyc (%.1f/mma)\n",
             mode ? "8-accumulators" : "1-accumulator", iters, h[0], (double)h[0] / iters, h[1],
             (double)h[1] / iters);
    }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
