// hmmaprobe.cu — throughput and latency of the warp-level tensor-core path
// (mma.sync.m16n8k16 f16 x f16 -> f32) on sm_100a, to size the warp-tile
// MLP kernel.  Each warp runs CH independent accumulator chains.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
template <int CH>
__global__ void tput(int iters, float* out, long long* cyc) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, 7u, 9u}, b[2] = {threadIdx.x ^ 5u, 3u};
  float d[CH][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) hmma(d[c], a, b);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int CH>
void run(int warps_per_sm, int sms) {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
  const int iters = 4096;
  tput<CH><<<sms, 32 * warps_per_sm>>>(16, o, c);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tput<CH><<<sms, 32 * warps_per_sm>>>(iters, o, c);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)sms * warps_per_sm * iters * CH * 16 * 8 * 16;
  printf("CH=%d warps/SM=%2d: %.1f TFLOP/s (%.0f MAC/clk/SM by clock64; %.1f cyc per HMMA per warp)\n", CH,
         warps_per_sm, 2 * macs / (ms * 1e-3) / 1e12, macs / sms / (double)cyc, (double)cyc / (iters * CH));
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1, 1); run<4>(1, 1); run<8>(1, 1);
  run<8>(4, 148); run<8>(8, 148); run<8>(16, 148); run<4>(32, 148); run<8>(32, 148);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
