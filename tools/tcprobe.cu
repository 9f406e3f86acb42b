// tcprobe.cu — on-device validation + microbenchmarks of the tcgen05 building
// blocks used by the fused query kernels (layouts of SMEM/TMEM operands,
// TMEM ld/st throughput, MMA round-trip latency).  Test tool, not product.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2305_02678_b200/csrc tools/tcprobe.cu -o tools/tcprobe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace nmq;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// A: [128][K] fp16 row-major in global, B: [N][K] fp16 row-major; D: [128][N] f32
// mode 0: A from SMEM; mode 1: A from TMEM (packed 2 fp16 per column)
template <int N, int K>
__global__ void mma_test(const __half* A, const __half* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  uint8_t* sA = smem;                       // K/8 chunks * 128 rows * 16 B
  uint8_t* sB = smem + (K / 8) * 128 * 16;  // K/8 chunks * N rows * 16 B
  // A rows: thread tid owns row tid
  for (int c = 0; c < K / 8; ++c) {
    const uint4 v = *reinterpret_cast<const uint4*>(A + tid * K + c * 8);
    *reinterpret_cast<uint4*>(sA + c * 128 * 16 + tid * 16) = v;
  }
  for (int i = tid; i < N * (K / 8); i += 128) {
    int n = i % N, c = i / N;
    const uint4 v = *reinterpret_cast<const uint4*>(B + n * K + c * 8);
    *reinterpret_cast<uint4*>(sB + c * N * 16 + n * 16) = v;
  }
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (tid < 32) tc::tmem_alloc<128>(&tbase);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t warp = tid / 32;
  const uint32_t lane_base = (warp * 32) << 16;
  const uint32_t a_col = 64;  // A in TMEM at columns [64, 64 + K/2)
  if (mode == 1) {
    // thread writes its row: column j holds (A[r][2j], A[r][2j+1])
    for (int j0 = 0; j0 < K / 2; j0 += 8) {
      uint32_t r[8];
      for (int j = 0; j < 8; ++j) {
        __half2 h = __halves2half2(A[tid * K + 2 * (j0 + j)], A[tid * K + 2 * (j0 + j) + 1]);
        r[j] = *reinterpret_cast<uint32_t*>(&h);
      }
      tc::tmem_st8(tb + lane_base + a_col + j0, r);
    }
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_f16(128, N);
    for (int s = 0; s < K / 16; ++s) {
      uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + s * 2 * N * 16, N * 16, 128);
      if (mode == 0) {
        uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + s * 2 * 128 * 16, 128 * 16, 128);
        tc::mma_ss(tb, ad, bd, idesc, s > 0);
      } else {
        tc::mma_ts(tb, tb + a_col + s * 8, bd, idesc, s > 0);
      }
    }
    tc::mma_commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    tc::tmem_ld8(tb + lane_base + c0, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 8; ++j) D[tid * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid < 32) tc::tmem_free<128>(tb);
}

// TMEM load throughput: each warp repeatedly loads x16 columns.
__global__ void ldtm_bench(int iters, float* sink, long long* cyc) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tc::tmem_alloc<128>(&tbase);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase + (((tid / 32) % 4 * 32) << 16);
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[16];
    tc::tmem_ld16(tb + ((i * 16) & 127), r);
    tc::tmem_ld_wait();
    #pragma unroll
    for (int j = 0; j < 16; ++j) acc += __uint_as_float(r[j]);
  }
  long long t1 = clock64();
  if (acc == 12345.f) sink[tid] = acc;
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid < 32) tc::tmem_free<128>(tbase);
}

// TMEM store throughput
__global__ void sttm_bench(int iters, long long* cyc) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tc::tmem_alloc<128>(&tbase);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase + (((tid / 32) % 4 * 32) << 16);
  uint32_t r[16];
  for (int j = 0; j < 16; ++j) r[j] = tid * 16 + j;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    r[0] += i;
    tc::tmem_st16(tb + ((i * 16) & 127), r);
  }
  tc::tmem_st_wait();
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid < 32) tc::tmem_free<128>(tbase);
}

// MMA round trip: issue K=16 x ksteps MMA (SS) + commit + all threads wait.
template <int N>
__global__ void mma_roundtrip(int iters, int ksteps, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < (16 * 1024) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
  if (tid < 32) tc::tmem_alloc<128>(&tbase);
  tc::fence_proxy_async_smem();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase;
  const uint32_t idesc = tc::idesc_f16(128, N);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (tid == 0) {
      for (int s = 0; s < ksteps; ++s) {
        uint64_t ad = tc::smem_desc(tc::smem_u32(smem) + (s & 3) * 4096, 2048, 128);
        uint64_t bd = tc::smem_desc(tc::smem_u32(smem) + 8192, N * 16, 128);
        tc::mma_ss(tb, ad, bd, idesc, s > 0);
      }
      tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, i & 1);
    tc::tc_fence_after();
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[blockIdx.x] = t1 - t0;
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid < 32) tc::tmem_free<128>(tb);
}

template <int N, int K>
int run_mma_test(int mode) {
  std::vector<__half> hA(128 * K), hB(N * K);
  std::vector<float> fA(128 * K), fB(N * K);
  srand(1234 + mode);
  for (int i = 0; i < 128 * K; ++i) { float v = (rand() % 17 - 8) / 8.0f; fA[i] = v; hA[i] = __float2half(v); }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 13 - 6) / 4.0f; fB[i] = v; hB[i] = __float2half(v); }
  __half *dA, *dB; float* dD;
  CK(cudaMalloc(&dA, hA.size() * 2)); CK(cudaMalloc(&dB, hB.size() * 2)); CK(cudaMalloc(&dD, 128 * N * 4));
  CK(cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemset(dD, 0, 128 * N * 4));
  int smem = (K / 8) * 128 * 16 + (K / 8) * N * 16;
  CK(cudaFuncSetAttribute(mma_test<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  mma_test<N, K><<<1, 128, smem>>>(dA, dB, dD, mode);
  CK(cudaDeviceSynchronize());
  std::vector<float> hD(128 * N);
  CK(cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int k = 0; k < K; ++k) ref += fA[m * K + k] * fB[n * K + k];
      if (std::fabs(ref - hD[m * N + n]) > 1e-3f) {
        if (bad < 6) printf("  mismatch m=%d n=%d got %f want %f\n", m, n, hD[m * N + n], ref);
        ++bad;
      }
    }
  printf("mma_test mode=%s N=%d K=%d: %s (%d bad)\n", mode ? "TS" : "SS", N, K, bad ? "FAIL" : "OK", bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad;
}

int main() {
  int bad = 0;
  bad += run_mma_test<32, 32>(0);
  bad += run_mma_test<16, 16>(0);
  bad += run_mma_test<16, 80>(0);
  bad += run_mma_test<32, 32>(1);
  bad += run_mma_test<16, 64>(1);
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs=%d clock(kHz)=%d\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  long long* dcyc; float* sink;
  CK(cudaMalloc(&dcyc, 4096 * 8)); CK(cudaMalloc(&sink, 4096 * 4));
  std::vector<long long> cyc(4096);
  // LDTM: 1 CTA of 128 threads and 1 CTA of 512 threads (16 warps) per SM
  for (int threads : {128, 256, 512}) {
    int iters = 4096;
    ldtm_bench<<<148, threads>>>(iters, sink, dcyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
    double bytes = (double)iters * threads * 16 * 4;
    printf("LDTM x16 threads/CTA=%d: %.1f cycles per warp-load, %.1f B/cycle/SM\n", threads,
           (double)cyc[0] / iters, bytes / cyc[0]);
    sttm_bench<<<148, threads>>>(iters, dcyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
    printf("STTM x16 threads/CTA=%d: %.1f cycles per warp-store, %.1f B/cycle/SM\n", threads,
           (double)cyc[0] / iters, bytes / cyc[0]);
  }
  for (int ks : {1, 2, 5}) {
    int iters = 2000;
    CK(cudaFuncSetAttribute(mma_roundtrip<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    mma_roundtrip<32><<<148, 128, 16384>>>(iters, ks, dcyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
    printf("MMA round trip N=32 ksteps=%d: %.1f cycles\n", ks, (double)cyc[0] / iters);
    CK(cudaFuncSetAttribute(mma_roundtrip<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    mma_roundtrip<16><<<148, 128, 16384>>>(iters, ks, dcyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
    printf("MMA round trip N=16 ksteps=%d: %.1f cycles\n", ks, (double)cyc[0] / iters);
  }
  // multiple CTAs per SM issuing round trips concurrently (throughput)
  for (int ctas : {4, 8}) {
    int iters = 2000;
    mma_roundtrip<32><<<148 * ctas, 128, 16384>>>(iters, 5, dcyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
    printf("MMA round trip N=32 ksteps=5, %d CTAs/SM: %.1f cycles per iter per CTA\n", ctas,
           (double)cyc[0] / iters);
  }
  printf("probe done, bad=%d\n", bad);
  return bad ? 1 : 0;
}
