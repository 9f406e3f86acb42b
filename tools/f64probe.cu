// Throughput probe (B200): F2F f32->f64, f64->f32, DFMA, DMUL, FFMA2, HADD2.F32 per SM per clock.
#include <cstdio>
#include <cuda_fp16.h>
#define N_ITER 4096
template <int OP>
__global__ void k(float* out, float s, long long* cyc) {
  float a = threadIdx.x * 1e-3f + s, b = a * 0.5f, c = a + 1.f, d = a - 1.f;
  double da = a, db = b, dc = c, dd = d;
  __half2 h = __floats2half2_rn(a, b);
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N_ITER; ++i) {
    if (OP == 0) {  // f32 -> f64 (4 independent)
      da += (double)a; db += (double)b; dc += (double)c; dd += (double)d;
      a = __int_as_float(__float_as_int(a) ^ 1); b = __int_as_float(__float_as_int(b) ^ 1);
    } else if (OP == 1) {  // DFMA
      da = fma(da, 1.0000001, 1e-9); db = fma(db, 1.0000001, 1e-9); dc = fma(dc, 1.0000001, 1e-9); dd = fma(dd, 1.0000001, 1e-9);
    } else if (OP == 2) {  // f64 -> f32
      a += (float)da; b += (float)db; c += (float)dc; d += (float)dd;
      da = __longlong_as_double(__double_as_longlong(da) ^ 1);
    } else if (OP == 3) {  // half -> float
      a += __low2float(h); b += __high2float(h); h = __hadd2(h, h);
    } else if (OP == 4) {  // FFMA
      a = fmaf(a, 1.0001f, 1e-3f); b = fmaf(b, 1.0001f, 1e-3f); c = fmaf(c, 1.0001f, 1e-3f); d = fmaf(d, 1.0001f, 1e-3f);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + (float)(da + db + dc + dd) + __low2float(h);
}
template <int OP>
void run(const char* name, int per_iter) {
  float* out; long long* cyc;
  int blocks = 148, threads = 1024;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  k<OP><<<blocks, threads>>>(out, 1.f, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, 1.f, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double ops = (double)threads * N_ITER * per_iter;  // per SM
  printf("%-12s %8.1f ops/clk/SM (thread-ops), %lld cycles\n", name, ops / c, c);
}
int main() {
  run<0>("f32->f64", 4); run<1>("DFMA", 4); run<2>("f64->f32", 4); run<3>("half->f32", 2); run<4>("FFMA", 4);
  return 0;
}
