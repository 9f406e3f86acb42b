// nmq_lod.cu — level of detail from ray cones, the step that produces the
// fractional lod the query kernels consume (render.py:334-337, 423-445).
// Float64 arithmetic like the reference (log2 of a squared footprint); the
// cone variant rounds the level to fp32, the lod type of the query API.
// HBM-bound elementwise kernels: 16-20 bytes per query, grid-stride loops
// over a multiple of the SM count.
#include <cstdint>
#include <cuda_runtime.h>
#include "nmq_internal.h"

namespace nmq {
namespace {

__device__ __forceinline__ double footprint_level(double area, double top) {
  // render.py:334-337: clip(0.5 * log2(max(area, 1)), 0, n_levels - 1)
  const double l = 0.5 * log2(fmax(area, 1.0));
  return fmin(fmax(l, 0.0), top);
}

__global__ void footprint_kernel(int64_t n, const double* __restrict__ area, double top,
                                 double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = footprint_level(__ldg(area + i), top);
}

// render.py:436-443: width = w + s t; diam = width / max(|cos|, 0.05); area = (diam * density)^2
__global__ void cone_kernel(int64_t n, const float* __restrict__ cone_w, const float* __restrict__ cone_s,
                            const float* __restrict__ t, const float* __restrict__ cos_hit,
                            const float* __restrict__ density, int32_t density_stride, double top,
                            float* __restrict__ lod) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double width = (double)__ldg(cone_w + i) + (double)__ldg(cone_s + i) * (double)__ldg(t + i);
    const double diam = width / fmax(fabs((double)__ldg(cos_hit + i)), 0.05);
    const double a = diam * (double)__ldg(density + i * density_stride);
    lod[i] = (float)footprint_level(a * a, top);
  }
}

int grid_for(int64_t n) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t want = (n + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(want < cap ? (want < 1 ? 1 : want) : cap);
}

}  // namespace

cudaError_t launch_footprint_level(int64_t n, const double* area, int32_t n_levels, double* out,
                                   cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  footprint_kernel<<<grid_for(n), 256, 0, s>>>(n, area, (double)(n_levels - 1), out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_cone_level(int64_t n, const float* cone_w, const float* cone_s, const float* t,
                              const float* cos_hit, const float* density, int32_t density_stride,
                              int32_t n_levels, float* lod, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cone_kernel<<<grid_for(n), 256, 0, s>>>(n, cone_w, cone_s, t, cos_hit, density, density_stride,
                                          (double)(n_levels - 1), lod);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace nmq
