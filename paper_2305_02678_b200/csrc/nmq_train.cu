// nmq_train.cu — training-side kernels: the exact adjoint of
// the latent fetch (latent.py:109-119 accumulate_texel_grads) and the fp32
// network engine's forward_cached / backward (mlp.py:90-116), used by the
// reference's offline baking loop (training.py).
//
//  * texel_grads_kernel: one thread per query — the same wrap-addressed taps
//    as the fetch (bit-exact indices), float64 bilinear weights like the
//    reference, contributions scattered with fp32 atomics into the gradient
//    texels (levels back to back, 8 channels).  Atomic/HBM-bound.
//  * mlp_forward_kernel: one thread per row, weights in SMEM, fp32 FMA (the
//    reference's float32 forward); pre-activations cached column-major
//    (coalesced per neuron) for the backward.
//  * mlp_backward_kernel: one thread per row, the reverse chain in float64
//    (the reference promotes to float64 at its first leaky layer), per-layer
//    output gradients cached column-major.
//  * mlp_dparam_kernel: dW = g^T x and db = sum g over the batch — a
//    split-K reduction: each CTA stages 32-row tiles of g and the layer
//    input (as float64) in SMEM, accumulates 4x4 register blocks of its
//    (out x in+1) partials in float64 and adds them to the result with
//    float64 atomics.
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <mutex>
#include "nmq_device.cuh"
#include "tc.cuh"
#include "nmq_internal.h"

namespace nmq {
namespace {

using namespace dev;

constexpr int kMaxW = 64;  // max layer width of the training kernels

// ---------------------------------------------------------------------------
// texel gradients

__device__ __forceinline__ void axis_f64(double c, int32_t n, int32_t& i0, int32_t& i1, double& f) {
  // latent.py:59-68: x = u*w - 0.5; x0 = floor(x) mod w (Python modulo); f = x - floor(x)
  const double fl = floor(c);
  f = c - fl;
  int64_t i = (int64_t)fl % n;
  if (i < 0) i += n;
  i0 = (int32_t)i;
  i1 = (i0 + 1 == n) ? 0 : i0 + 1;
}

// The coarse tail of the pyramid (levels of <= 16x16 texels, a few hundred
// texels) receives a large share of all taps — with a uniform lod every level
// takes 1/L of the queries, the 1x1 level all 4 taps of each — so its
// contributions are pre-summed per CTA in SMEM and flushed once (global
// atomics on those addresses serialised at L2 dominated the scatter).
constexpr int kTailTexels = 512;

__global__ void texel_grads_kernel(const __grid_constant__ MatParams mp, int64_t n,
                                   const float* __restrict__ uv, const int32_t* __restrict__ level,
                                   const float* __restrict__ z_grad, float* __restrict__ grad,
                                   bool vec, int64_t tail_start, int tail_n) {
  __shared__ __align__(16) float tail[kTailTexels * 8];
  for (int i = threadIdx.x; i < tail_n * 8; i += blockDim.x) tail[i] = 0.f;
  __syncthreads();
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    int l = __ldg(level + q);
    l = l < 0 ? 0 : (l > mp.n_levels - 1 ? mp.n_levels - 1 : l);
    const LevelDesc L = mp.lv[l];
    int32_t x0, x1, y0, y1;
    double fx, fy;
    axis_f64(fma((double)__ldg(uv + 2 * q), (double)L.w, -0.5), L.w, x0, x1, fx);
    axis_f64(fma((double)__ldg(uv + 2 * q + 1), (double)L.h, -0.5), L.h, y0, y1, fy);
    const double w[4] = {(1.0 - fx) * (1.0 - fy), fx * (1.0 - fy), (1.0 - fx) * fy, fx * fy};
    const int32_t xs[4] = {x0, x1, x0, x1}, ys[4] = {y0, y0, y1, y1};  // latent.py:69-73 tap order
    float g[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) g[c] = __ldg(z_grad + 8 * q + c);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t t = L.off + (int64_t)ys[k] * L.w + xs[k];
      float v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = (float)(w[k] * (double)g[c]);
      if (t >= tail_start) {
#pragma unroll
        for (int c = 0; c < 8; ++c) atomicAdd(tail + 8 * (t - tail_start) + c, v[c]);
      } else if (vec) {  // two 16-byte vector reductions per texel (same fp32 atomic adds)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(grad + 8 * t + 4 * h),
                       "f"(v[4 * h]), "f"(v[4 * h + 1]), "f"(v[4 * h + 2]), "f"(v[4 * h + 3])
                       : "memory");
      } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) atomicAdd(grad + 8 * t + c, v[c]);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < tail_n; i += blockDim.x) {
    const float4 lo = reinterpret_cast<const float4*>(tail)[2 * i];
    const float4 hi = reinterpret_cast<const float4*>(tail)[2 * i + 1];
    const bool touched = lo.x != 0.f || lo.y != 0.f || lo.z != 0.f || lo.w != 0.f || hi.x != 0.f ||
                         hi.y != 0.f || hi.z != 0.f || hi.w != 0.f;
    if (!touched) continue;
    float* dst = grad + 8 * (tail_start + i);
    if (vec) {
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(lo.x), "f"(lo.y),
                   "f"(lo.z), "f"(lo.w) : "memory");
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4), "f"(hi.x), "f"(hi.y),
                   "f"(hi.z), "f"(hi.w) : "memory");
    } else {
      const float v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int c = 0; c < 8; ++c) atomicAdd(dst + c, v[c]);
    }
  }
}

// ---------------------------------------------------------------------------
// MLP forward_cached / backward

struct MlpView {
  int32_t n_layers;
  int32_t fi[kMaxLayers], fo[kMaxLayers], act[kMaxLayers];
  int32_t w_off[kMaxLayers];  // float offset of layer l in the access-order weights
  int32_t w_floats;
  int32_t p_off[kMaxLayers];  // forward (kPad): layer offsets of the padded SMEM copy
};

// kPad: every weight row zero-padded to kMW (+ the bias at index kMW, rows
// 16-byte aligned) and activations zero beyond the layer width, so the inner
// product runs unpredicated over kMW with LDS.128 weight reads; the appended
// terms are 0 * 0, so each row's fp32 FMA chain is unchanged (the per-k
// predicates of the unpadded instance cost as many ISETPs as FFMAs).
template <int kMW, bool kPad>
__global__ void mlp_forward_kernel(const __grid_constant__ MlpView v, int64_t B,
                                   const float* __restrict__ wts, const float* __restrict__ x,
                                   float* __restrict__ x_cache, float* __restrict__ pre_cache,
                                   float* __restrict__ out) {
  extern __shared__ float4 sw4[];
  float* sw = reinterpret_cast<float*>(sw4);
  constexpr int rs = kMW + 4;
  if (kPad) {
    for (int l = 0; l < v.n_layers; ++l) {
      const int fi = v.fi[l];
      const float* wl = wts + v.w_off[l];
      for (int i = threadIdx.x; i < v.fo[l] * rs; i += blockDim.x) {
        const int j = i / rs, k = i % rs;
        sw[v.p_off[l] + i] = k < fi ? wl[j * (fi + 1) + k] : (k == kMW ? wl[j * (fi + 1) + fi] : 0.f);
      }
    }
  } else {
    for (int i = threadIdx.x; i < v.w_floats; i += blockDim.x) sw[i] = wts[i];
  }
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < B;
       r += (int64_t)gridDim.x * blockDim.x) {
    float a[kMW], p[kMW];
    const int fi0 = v.fi[0];
#pragma unroll
    for (int k = 0; k < kMW; ++k) {
      if (k < fi0) {
        a[k] = __ldg(x + r * fi0 + k);
        x_cache[(int64_t)k * B + r] = a[k];
      } else {
        a[k] = 0.f;
      }
    }
    int64_t pre_base = 0;
    for (int l = 0; l < v.n_layers; ++l) {
      const int fi = v.fi[l], fo = v.fo[l];
      if (kPad) {
        const float* W = sw + v.p_off[l];
#pragma unroll
        for (int j = 0; j < kMW; ++j) {
          if (j < fo) {
            const float4* row = reinterpret_cast<const float4*>(W + j * rs);
            float acc = 0.f;
#pragma unroll
            for (int k4 = 0; k4 < kMW / 4; ++k4) {
              const float4 w = row[k4];
              acc = fmaf(a[4 * k4 + 0], w.x, acc);
              acc = fmaf(a[4 * k4 + 1], w.y, acc);
              acc = fmaf(a[4 * k4 + 2], w.z, acc);
              acc = fmaf(a[4 * k4 + 3], w.w, acc);
            }
            p[j] = acc + W[j * rs + kMW];  // x W^T + b (mlp.py:96)
            pre_cache[pre_base + (int64_t)j * B + r] = p[j];
          } else {
            p[j] = 0.f;  // keeps the next layer's padded inputs zero
          }
        }
      } else {
        const float* W = sw + v.w_off[l];
#pragma unroll
        for (int j = 0; j < kMW; ++j) {
          if (j < fo) {
            const float* row = W + j * (fi + 1);
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < kMW; ++k)
              if (k < fi) acc = fmaf(a[k], row[k], acc);
            p[j] = acc + row[fi];  // x W^T + b (mlp.py:96)
            pre_cache[pre_base + (int64_t)j * B + r] = p[j];
          }
        }
      }
      const bool leaky = v.act[l] != 0;
#pragma unroll
      for (int j = 0; j < kMW; ++j)
        if (kPad || j < fo) a[j] = leaky ? (p[j] >= 0.f ? p[j] : kLeaky * p[j]) : p[j];
      pre_base += (int64_t)fo * B;
    }
    const int fl = v.fo[v.n_layers - 1];
#pragma unroll
    for (int j = 0; j < kMW; ++j)
      if (j < fl) out[r * fl + j] = a[j];
  }
}

template <int kMW, typename WT>
__global__ void mlp_backward_kernel(const __grid_constant__ MlpView v, int64_t B,
                                    const float* __restrict__ wts, const float* __restrict__ pre_cache,
                                    const float* __restrict__ out_grad, double* __restrict__ g_cache,
                                    double* __restrict__ dx) {
  // WT = double: weights widened to float64 once at staging (exact), so the
  // chain's DFMAs take them straight from SMEM without a per-use F2F
  // conversion; WT = float for networks whose float64 copy exceeds SMEM
  extern __shared__ __align__(8) unsigned char sraw[];
  WT* swd = reinterpret_cast<WT*>(sraw);
  for (int i = threadIdx.x; i < v.w_floats; i += blockDim.x) swd[i] = (WT)wts[i];
  __syncthreads();
  int64_t pre_off[kMaxLayers];
  {
    int64_t o = 0;
    for (int l = 0; l < v.n_layers; ++l) {
      pre_off[l] = o;
      o += (int64_t)v.fo[l] * B;
    }
  }
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < B;
       r += (int64_t)gridDim.x * blockDim.x) {
    // one register array: the layer's output gradient goes to g_cache (which
    // the dW/db reduction needs anyway) and is read back from there (L1) for
    // g @ W, so g and g @ W are never live at once (half the registers)
    double g[kMW];
    const int fl = v.fo[v.n_layers - 1];
#pragma unroll
    for (int j = 0; j < kMW; ++j)
      if (j < fl) g[j] = (double)__ldg(out_grad + r * fl + j);
    for (int l = v.n_layers - 1; l >= 0; --l) {
      const int fi = v.fi[l], fo = v.fo[l];
      const bool leaky = v.act[l] != 0;
      double* gc = g_cache + pre_off[l] + r;
#pragma unroll
      for (int j = 0; j < kMW; ++j) {
        if (j < fo) {
          if (leaky && __ldg(pre_cache + pre_off[l] + (int64_t)j * B + r) < 0.f) g[j] *= (double)kLeaky;
          gc[(int64_t)j * B] = g[j];  // same column-major layout as pre
        }
      }
      const WT* W = swd + v.w_off[l];
#pragma unroll
      for (int k = 0; k < kMW; ++k) g[k] = 0.0;
      for (int j = 0; j < fo; ++j) {  // g @ W (mlp.py:115), same j order per element
        const double gj = gc[(int64_t)j * B];
        const WT* Wj = W + j * (fi + 1);
#pragma unroll
        for (int k = 0; k < kMW; ++k)
          if (k < fi) g[k] = fma(gj, (double)Wj[k], g[k]);
      }
    }
    const int fi0 = v.fi[0];
#pragma unroll
    for (int k = 0; k < kMW; ++k)
      if (k < fi0) dx[r * fi0 + k] = g[k];
  }
}

// dW[j][k] = sum_r g[j][r] * in[k][r], db[j] = sum_r g[j][r]   (mlp.py:114)
// `in` = the cached input x (layer 0) or act(pre of the previous layer).
constexpr int kRowsPerCta = 256, kTileRows = 32;  // B/256 CTAs of split-K partials per layer

// Register-blocked: a thread owns a 4(j) x 4(k) block of (dW | db) and reads
// its 4 g and 4 inputs per row as two 16-byte SMEM loads each (inputs are
// converted to float64 once, at staging), 16 DFMA per 4 loads.  Narrow layers
// (< 128 blocks) split the tile rows over R thread slices whose partials meet
// in a float64 SMEM reduction before the one global atomic per parameter.
constexpr int kBlk = 4;

struct DparamArgs {  // every layer of one network: blockIdx.y = layer
  int32_t fi[kMaxLayers], fo[kMaxLayers], in_act[kMaxLayers];
  const float* in_src[kMaxLayers];
  const double* g[kMaxLayers];
  double* dp[kMaxLayers];
};

// kMW = the network's widest layer (32 or 64): sizes the register blocks,
// prefetch registers and SMEM (the 32-wide instance fits 3 CTAs per SM)
template <int kMW>
__global__ void __launch_bounds__(256) mlp_dparam_kernel(const __grid_constant__ DparamArgs args, int64_t B) {
  constexpr int kMaxNbJ = (kMW + kBlk - 1) / kBlk, kMaxNbK = (kMW + 1 + kBlk - 1) / kBlk;
  constexpr int kBlkPer = (kMaxNbJ * kMaxNbK + 255) / 256;
  constexpr int kGPer = (kBlk * kMaxNbJ * kTileRows + 255) / 256;
  constexpr int kXPer = (kBlk * kMaxNbK * kTileRows + 255) / 256;
  constexpr int kDpSmem = kTileRows * (kBlk * kMaxNbJ + 2) + kTileRows * (kBlk * kMaxNbK + 2);
  static_assert(kDpSmem >= kMW * (kMW + 1), "reduction buffer reuses the staging tiles");
  const int l = blockIdx.y;
  const int fi = args.fi[l], fo = args.fo[l], in_act = args.in_act[l];
  const float* __restrict__ in_src = args.in_src[l];
  const double* __restrict__ g = args.g[l];
  double* __restrict__ dp = args.dp[l];
  __shared__ __align__(16) double smem[kDpSmem];
  const int njb = (fo + kBlk - 1) / kBlk, nkb = (fi + 1 + kBlk - 1) / kBlk, nb = njb * nkb;
  // row strides padded by 2 doubles (16-byte aligned rows, fewer store conflicts)
  const int SJ = kBlk * njb + 2, SK = kBlk * nkb + 2;
  double* sg = smem;                  // [kTileRows][SJ]
  double* sx = smem + kTileRows * SJ;  // [kTileRows][SK]
  const int R = nb >= 128 ? 1 : (256 / nb < kTileRows ? 256 / nb : kTileRows);
  const int t = threadIdx.x;
  double acc[kBlkPer][kBlk * kBlk];
#pragma unroll
  for (int e = 0; e < kBlkPer; ++e)
#pragma unroll
    for (int i = 0; i < kBlk * kBlk; ++i) acc[e][i] = 0.0;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta;
  const int64_t r1 = r0 + kRowsPerCta < B ? r0 + kRowsPerCta : B;
  // the next tile's g and inputs are loaded into registers while the current
  // one is reduced (17 loads in flight per thread instead of one)
  const int ng = kBlk * njb * kTileRows, nx = kBlk * nkb * kTileRows;
  double gr[kGPer];
  float xr[kXPer];
  auto load = [&](int64_t t0) {
#pragma unroll
    for (int u = 0; u < kGPer; ++u) {
      const int i = t + u * 256, j = i / kTileRows;
      if (i >= ng) break;  // warp-uniform (ng is a multiple of 128): narrow layers skip the rest
      const int64_t r = t0 + i % kTileRows;
      gr[u] = (j < fo && r < r1) ? g[(int64_t)j * B + r] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kXPer; ++u) {
      const int i = t + u * 256, k = i / kTileRows;
      if (i >= nx) break;
      const int64_t r = t0 + i % kTileRows;
      float xv = 0.f;
      if (r < r1 && k <= fi) {
        if (k == fi) {
          xv = 1.f;  // bias column
        } else {
          xv = in_src[(int64_t)k * B + r];
          if (in_act && xv < 0.f) xv *= kLeaky;
        }
      }
      xr[u] = xv;
    }
  };
  load(r0);
  for (int64_t t0 = r0; t0 < r1; t0 += kTileRows) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kGPer; ++u) {
      const int i = t + u * 256;
      if (i >= ng) break;
      sg[(i % kTileRows) * SJ + i / kTileRows] = gr[u];
    }
#pragma unroll
    for (int u = 0; u < kXPer; ++u) {
      const int i = t + u * 256;
      if (i >= nx) break;
      sx[(i % kTileRows) * SK + i / kTileRows] = (double)xr[u];
    }
    __syncthreads();
    if (t0 + kTileRows < r1) load(t0 + kTileRows);
#pragma unroll
    for (int e = 0; e < kBlkPer; ++e) {
      const int blk = R > 1 ? t % nb : t + e * 256;
      const int slice = R > 1 ? t / nb : 0;
      if ((R > 1 && (e > 0 || slice >= R)) || blk >= nb) continue;
      const double* gp = sg + kBlk * (blk / nkb);
      const double* xp = sx + kBlk * (blk % nkb);
      for (int rr = slice; rr < kTileRows; rr += R) {
        const double2 g01 = *reinterpret_cast<const double2*>(gp + rr * SJ);
        const double2 g23 = *reinterpret_cast<const double2*>(gp + rr * SJ + 2);
        const double2 x01 = *reinterpret_cast<const double2*>(xp + rr * SK);
        const double2 x23 = *reinterpret_cast<const double2*>(xp + rr * SK + 2);
        const double gv[4] = {g01.x, g01.y, g23.x, g23.y}, xv[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
        for (int a = 0; a < kBlk; ++a)
#pragma unroll
          for (int c = 0; c < kBlk; ++c) acc[e][a * kBlk + c] = fma(gv[a], xv[c], acc[e][a * kBlk + c]);
      }
    }
  }
  const int pairs = fo * (fi + 1);
  if (R > 1) {  // slices meet in SMEM, then one global atomic per parameter
    __syncthreads();
    for (int i = t; i < pairs; i += blockDim.x) smem[i] = 0.0;
    __syncthreads();
  }
#pragma unroll
  for (int e = 0; e < kBlkPer; ++e) {
    const int blk = R > 1 ? t % nb : t + e * 256;
    const int slice = R > 1 ? t / nb : 0;
    if ((R > 1 && (e > 0 || slice >= R)) || blk >= nb) continue;
    const int j0 = kBlk * (blk / nkb), k0 = kBlk * (blk % nkb);
#pragma unroll
    for (int a = 0; a < kBlk; ++a)
#pragma unroll
      for (int c = 0; c < kBlk; ++c) {
        const int j = j0 + a, k = k0 + c;
        if (j < fo && k <= fi) {
          if (R > 1) atomicAdd(smem + j * (fi + 1) + k, acc[e][a * kBlk + c]);
          else atomicAdd(dp + j * (fi + 1) + k, acc[e][a * kBlk + c]);
        }
      }
  }
  if (R > 1) {
    __syncthreads();
    for (int i = t; i < pairs; i += blockDim.x) atomicAdd(dp + i, smem[i]);
  }
}

// ---------------------------------------------------------------------------
// dW / db on the tensor cores (tcgen05.mma kind::tf32), 3xTF32: every operand
// is split a = hi + lo (hi = a with its low 13 mantissa bits cleared, exact
// in tf32; lo = a - hi, whose own tf32 truncation keeps ~11 more bits) and
// D += A_hi B_hi + A_hi B_lo + A_lo B_hi — each product to ~2^-21 relative,
// fp32 accumulation in TMEM over one CTA's rows, float64 atomics across
// CTAs.  A = g^T (M = 128 >= fo rows, K = batch: g is cached column-major,
// so K is contiguous), B = [x | 1] (N = fi + 1 padded to 16, K = batch), both
// K-major in SMEM in the canonical no-swizzle layout: element (row, k) at
// (k / 4) * (rows * 16) + row * 16 + (k % 4) * 4 — 8-row x 16-byte core
// matrices, SBO = 128 B between row groups, LBO = rows * 16 B between k
// chunks.  The reference's float64 chain is replaced only in this reduction
// (parity: tests/test_gpu_parity.py::test_mlp_forward_cached_backward_*).
#ifndef NMQ_TC_KT
#define NMQ_TC_KT 32
#endif
#ifndef NMQ_TC_ROWS
#define NMQ_TC_ROWS 256
#endif
constexpr int kTcM = 128, kTcNMax = 80, kTcKT = NMQ_TC_KT, kTcRows = NMQ_TC_ROWS;  // rows per CTA (split-K)
constexpr size_t kTcSmem = (size_t)2 * (kTcM + kTcNMax) * kTcKT * 4;

__device__ __forceinline__ void split_tf32(float v, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  lo = v - hi;  // exact
}

__global__ void __launch_bounds__(128) mlp_dparam_tc_kernel(const __grid_constant__ DparamArgs args, int64_t B) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_sh;
  const int l = blockIdx.y;
  const int fi = args.fi[l], fo = args.fo[l], in_act = args.in_act[l];
  const float* __restrict__ in_src = args.in_src[l];
  const double* __restrict__ g = args.g[l];
  double* __restrict__ dp = args.dp[l];
  const int np = ((fi + 1) + 15) / 16 * 16;  // N: inputs + the bias column, padded
  float* a_hi = reinterpret_cast<float*>(sm);
  float* a_lo = a_hi + kTcM * kTcKT;
  float* b_hi = a_lo + kTcM * kTcKT;
  float* b_lo = b_hi + kTcNMax * kTcKT;
  const int t = threadIdx.x, warp = t / 32;
  auto off = [](int rows, int row, int k) { return (k >> 2) * (rows * 4) + row * 4 + (k & 3); };  // in floats
  // padded rows stay zero: A rows >= fo, B rows > fi
  for (int i = t; i < (int)(kTcSmem / 4); i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (t == 0) tc::mbar_init(&bar, 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(tc::smem_u32(&tbase_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_mbar_init();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase_sh;
  const int64_t r0 = (int64_t)blockIdx.x * kTcRows;
  const int64_t r1 = r0 + kTcRows < B ? r0 + kTcRows : B;
  constexpr uint32_t idesc = tc::idesc_tf32(kTcM, 16);  // N patched below (runtime)
  const uint32_t id = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(np >> 3) << 17);
  // the next tile's g and inputs are loaded into registers while the tensor
  // core runs the current one (consecutive threads take consecutive k of one
  // row: coalesced)
  constexpr int kGPer = kMaxW * kTcKT / 128, kXPer = (kMaxW + 1) * kTcKT / 128 + 1;
  double gr[kGPer];
  float xr[kXPer];
  const int ng = fo * kTcKT, nx = (fi + 1) * kTcKT;
  auto load = [&](int64_t t0) {
#pragma unroll
    for (int u = 0; u < kGPer; ++u) {
      const int i = t + 128 * u;
      if (i >= ng) break;
      const int m = i / kTcKT, k = i % kTcKT;
      gr[u] = t0 + k < r1 ? g[(int64_t)m * B + t0 + k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kXPer; ++u) {
      const int i = t + 128 * u;
      if (i >= nx) break;
      const int n = i / kTcKT, k = i % kTcKT;
      float xv = 0.f;
      if (t0 + k < r1) {
        if (n == fi) {
          xv = 1.f;  // bias column: db = sum g
        } else {
          xv = in_src[(int64_t)n * B + t0 + k];
          if (in_act && xv < 0.f) xv *= kLeaky;
        }
      }
      xr[u] = xv;
    }
  };
  load(r0);
  uint32_t phase = 0;
  for (int64_t t0 = r0; t0 < r1; t0 += kTcKT) {
#pragma unroll
    for (int u = 0; u < kGPer; ++u) {
      const int i = t + 128 * u;
      if (i >= ng) break;
      const int m = i / kTcKT, k = i % kTcKT;
      const double v = gr[u];
      const float hi = __uint_as_float(__float_as_uint((float)v) & 0xFFFFE000u);
      a_hi[off(kTcM, m, k)] = hi;
      a_lo[off(kTcM, m, k)] = (float)(v - (double)hi);
    }
#pragma unroll
    for (int u = 0; u < kXPer; ++u) {
      const int i = t + 128 * u;
      if (i >= nx) break;
      const int n = i / kTcKT, k = i % kTcKT;
      float hi, lo;
      split_tf32(xr[u], hi, lo);
      b_hi[off(kTcNMax, n, k)] = hi;
      b_lo[off(kTcNMax, n, k)] = lo;
    }
    tc::fence_proxy_async_smem();  // generic-proxy stores -> the tensor core's async proxy
    tc::tc_fence_before();
    __syncthreads();
    if (t == 0) {
      tc::tc_fence_after();
      const uint32_t lbo_a = kTcM * 16, lbo_b = kTcNMax * 16;
#pragma unroll
      for (int s = 0; s < kTcKT / 8; ++s) {  // K = 8 tf32 = 2 k-chunks per MMA
        const uint64_t ah = tc::smem_desc(tc::smem_u32(a_hi) + 2 * s * lbo_a, lbo_a, 128);
        const uint64_t al = tc::smem_desc(tc::smem_u32(a_lo) + 2 * s * lbo_a, lbo_a, 128);
        const uint64_t bh = tc::smem_desc(tc::smem_u32(b_hi) + 2 * s * lbo_b, lbo_b, 128);
        const uint64_t bl = tc::smem_desc(tc::smem_u32(b_lo) + 2 * s * lbo_b, lbo_b, 128);
        tc::mma_ss_tf32(tb, ah, bh, id, (t0 > r0 || s > 0) ? 1u : 0u);
        tc::mma_ss_tf32(tb, ah, bl, id, 1u);
        tc::mma_ss_tf32(tb, al, bh, id, 1u);
      }
      tc::mma_commit(&bar);
    }
    if (t0 + kTcKT < r1) load(t0 + kTcKT);
    tc::mbar_wait(&bar, phase);  // the MMAs have read the tile before it is overwritten
    phase ^= 1u;
    tc::tc_fence_after();
  }
  // row m of D (TMEM lane m) -> dW[m][0..fi], db[m] = column fi
  const int m = t;
  const uint32_t lane_addr = tb + ((uint32_t)(warp * 32) << 16);
  for (int c0 = 0; c0 < np; c0 += 16) {
    uint32_t r[16];
    tc::tmem_ld16(lane_addr + (uint32_t)c0, r);
    tc::tmem_ld_wait();
    if (m < fo) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j <= fi) atomicAdd(dp + (int64_t)m * (fi + 1) + c0 + j, (double)__uint_as_float(r[j]));
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb) : "memory");
}

// The same reduction fed by 2-D TMA: each layer's g (fo x B, float64) and
// input (fi x B, fp32) caches are tensor maps; one box load per operand
// brings a 32-row tile ([fo][32] / [fi][32], zero-filled past B) into a
// 3-stage SMEM ring; all threads split the tile into the tf32 hi / lo operand
// layout of one of two buffers while the tensor core runs on the other.
// ~One CTA per SM over all layers.
constexpr int kTmS = 3, kTmKT = 32, kTmThreads = 256, kTmFlush = 8;  // flush D every 8 tiles = 256 rows
constexpr size_t kTmRawG = (size_t)kMaxW * kTmKT * 8, kTmRawX = (size_t)kMaxW * kTmKT * 4;
constexpr size_t kTmSplit = (size_t)2 * (kTcM + kTcNMax) * kTmKT * 4;
constexpr size_t kTmSmem = kTmS * (kTmRawG + kTmRawX) + 2 * kTmSplit + 128;  // + alignment slack

struct DparamMaps {
  CUtensorMap g[kMaxLayers], x[kMaxLayers];
};

__global__ void __launch_bounds__(kTmThreads) mlp_dparam_tma_kernel(const __grid_constant__ DparamArgs args,
                                                                    const __grid_constant__ DparamMaps maps,
                                                                    int64_t B, int64_t rows_per_cta) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>(((uintptr_t)sm_raw + 127) & ~(uintptr_t)127);  // TMA: 128-B aligned
  __shared__ uint64_t full[kTmS], mma_done[2];
  __shared__ uint32_t tbase_sh;
  const int l = blockIdx.y;
  const int fi = args.fi[l], fo = args.fo[l], in_act = args.in_act[l];
  double* __restrict__ dp = args.dp[l];
  const int np = ((fi + 1) + 15) / 16 * 16;
  const int t = threadIdx.x, warp = t / 32;
  uint8_t* raw = sm;
  uint8_t* split = sm + kTmS * (kTmRawG + kTmRawX);
  auto raw_g = [&](int st) { return reinterpret_cast<double*>(raw + st * (kTmRawG + kTmRawX)); };
  auto raw_x = [&](int st) { return reinterpret_cast<float*>(raw + st * (kTmRawG + kTmRawX) + kTmRawG); };
  auto off = [](int rows, int row, int k) { return (k >> 2) * (rows * 4) + row * 4 + (k & 3); };
  for (int i = t; i < (int)(2 * kTmSplit / 4); i += kTmThreads) reinterpret_cast<float*>(split)[i] = 0.f;
  if (t == 0) {
    for (int i = 0; i < kTmS; ++i) tc::mbar_init(&full[i], 1);
    tc::mbar_init(&mma_done[0], 1);
    tc::mbar_init(&mma_done[1], 1);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(tc::smem_u32(&tbase_sh))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_mbar_init();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase_sh;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = r0 + rows_per_cta < B ? r0 + rows_per_cta : B;
  const int ntile = r1 > r0 ? (int)((r1 - r0 + kTmKT - 1) / kTmKT) : 0;
  const uint32_t box_bytes = (uint32_t)kTmKT * (8u * fo + 4u * fi);
  auto issue = [&](int j) {  // thread 0
    const int st = j % kTmS;
    const int32_t t0 = (int32_t)(r0 + (int64_t)j * kTmKT);
    tc::mbar_arrive_expect_tx(&full[st], box_bytes);
    tc::tma_load_2d(tc::smem_u32(raw_g(st)), &maps.g[l], t0, 0, &full[st]);
    if (fi > 0) tc::tma_load_2d(tc::smem_u32(raw_x(st)), &maps.x[l], t0, 0, &full[st]);
  };
  if (t == 0)
    for (int j = 0; j < kTmS && j < ntile; ++j) issue(j);
  const uint32_t id = (tc::idesc_tf32(kTcM, 16) & ~(0x3Fu << 17)) | ((uint32_t)(np >> 3) << 17);
  // D (fp32 in TMEM) is flushed into the float64 result every kTmFlush tiles,
  // so fp32 accumulates over at most 256 rows whatever the batch
  auto flush = [&]() {
    if (warp < 4) {  // warps 0-3 own TMEM lanes 0-127 (D row = lane)
      const uint32_t lane_addr = tb + ((uint32_t)(warp * 32) << 16);
      for (int c0 = 0; c0 < np; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(lane_addr + (uint32_t)c0, r);
        tc::tmem_ld_wait();
        if (t < fo) {
#pragma unroll
          for (int q = 0; q < 16; ++q)
            if (c0 + q <= fi) atomicAdd(dp + (int64_t)t * (fi + 1) + c0 + q, (double)__uint_as_float(r[q]));
        }
      }
    }
  };
  int acc_from = 0;  // first tile of the current fp32 accumulation
  for (int j = 0; j < ntile; ++j) {
    const int st = j % kTmS, b = j & 1;
    const int64_t t0 = r0 + (int64_t)j * kTmKT;
    const int rows = (int)(r1 - t0 < kTmKT ? r1 - t0 : kTmKT);  // rows past r1 (but < B) are another CTA's
    tc::mbar_wait(&full[st], (uint32_t)(j / kTmS) & 1u);
    if (j >= 2) tc::mbar_wait(&mma_done[b], (uint32_t)((j - 2) / 2) & 1u);  // buffer b's MMAs are done
    tc::tc_fence_after();
    float* a_hi = reinterpret_cast<float*>(split + b * kTmSplit);
    float* a_lo = a_hi + kTcM * kTmKT;
    float* b_hi = a_lo + kTcM * kTmKT;
    float* b_lo = b_hi + kTcNMax * kTmKT;
    const double* rg = raw_g(st);
    const float* rx = raw_x(st);
    // one item = one row x 4 consecutive k (the box is dense: [row][32])
    for (int i = t; i < fo * (kTmKT / 4); i += kTmThreads) {
      const int m = i / (kTmKT / 4), k0 = 4 * (i % (kTmKT / 4));
      const double2 v01 = *reinterpret_cast<const double2*>(rg + m * kTmKT + k0);
      const double2 v23 = *reinterpret_cast<const double2*>(rg + m * kTmKT + k0 + 2);
      const double v[4] = {k0 < rows ? v01.x : 0.0, k0 + 1 < rows ? v01.y : 0.0, k0 + 2 < rows ? v23.x : 0.0,
                           k0 + 3 < rows ? v23.y : 0.0};
      float hi[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hi[q] = __uint_as_float(__float_as_uint((float)v[q]) & 0xFFFFE000u);
        lo[q] = (float)(v[q] - (double)hi[q]);
      }
      *reinterpret_cast<float4*>(a_hi + off(kTcM, m, k0)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(a_lo + off(kTcM, m, k0)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
    for (int i = t; i < (fi + 1) * (kTmKT / 4); i += kTmThreads) {
      const int n = i / (kTmKT / 4), k0 = 4 * (i % (kTmKT / 4));
      float xv[4] = {1.f, 1.f, 1.f, 1.f};  // bias column: db = sum g
      if (n < fi) {
        const float4 r4 = *reinterpret_cast<const float4*>(rx + n * kTmKT + k0);
        xv[0] = r4.x; xv[1] = r4.y; xv[2] = r4.z; xv[3] = r4.w;
        if (in_act) {
#pragma unroll
          for (int q = 0; q < 4; ++q) xv[q] = xv[q] < 0.f ? xv[q] * kLeaky : xv[q];
        }
      }
      float hi[4], lo[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) split_tf32(k0 + q < rows ? xv[q] : 0.f, hi[q], lo[q]);
      *reinterpret_cast<float4*>(b_hi + off(kTcNMax, n, k0)) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4*>(b_lo + off(kTcNMax, n, k0)) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
    tc::fence_proxy_async_smem();  // the split tile -> the tensor core's async proxy
    tc::tc_fence_before();
    __syncthreads();               // raw stage st fully read; split buffer b complete
    if (t == 0) {
      tc::tc_fence_after();
      const uint32_t lbo_a = kTcM * 16, lbo_b = kTcNMax * 16;
#pragma unroll
      for (int s2 = 0; s2 < kTmKT / 8; ++s2) {
        const uint64_t ah = tc::smem_desc(tc::smem_u32(a_hi) + 2 * s2 * lbo_a, lbo_a, 128);
        const uint64_t al = tc::smem_desc(tc::smem_u32(a_lo) + 2 * s2 * lbo_a, lbo_a, 128);
        const uint64_t bh = tc::smem_desc(tc::smem_u32(b_hi) + 2 * s2 * lbo_b, lbo_b, 128);
        const uint64_t bl = tc::smem_desc(tc::smem_u32(b_lo) + 2 * s2 * lbo_b, lbo_b, 128);
        tc::mma_ss_tf32(tb, ah, bh, id, (j > acc_from || s2 > 0) ? 1u : 0u);
        tc::mma_ss_tf32(tb, ah, bl, id, 1u);
        tc::mma_ss_tf32(tb, al, bh, id, 1u);
      }
      tc::mma_commit(&mma_done[b]);
      if (j + kTmS < ntile) issue(j + kTmS);  // refill the stage just consumed
    }
    if ((j + 1) % kTmFlush == 0 && j + 1 < ntile) {
      tc::mbar_wait(&mma_done[b], (uint32_t)(j / 2) & 1u);
      tc::tc_fence_after();
      flush();
      tc::tc_fence_before();
      __syncthreads();  // D read before the next tile's first MMA overwrites it
      acc_from = j + 1;
    }
  }
  if (ntile > 0) {
    const int jl = ntile - 1;
    tc::mbar_wait(&mma_done[jl & 1], (uint32_t)(jl / 2) & 1u);
    tc::tc_fence_after();
    flush();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb) : "memory");
}

PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(p);
  });
  return fn;
}

// [rows][B] row-major cache (row stride B elements) as a 2-D tensor map with
// box [rows][kTmKT]
bool encode_rows(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize, int64_t B, int rows) {
  PFN_cuTensorMapEncodeTiled fn = encode_fn();
  if (!fn || rows < 1 || rows > 256 || ((uintptr_t)base & 15u) || (B * esize) % 16) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)(B * esize)};
  const cuuint32_t box[2] = {(cuuint32_t)kTmKT, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int max_width(const MlpView& v) {
  int w = 0;
  for (int l = 0; l < v.n_layers; ++l) {
    w = v.fi[l] > w ? v.fi[l] : w;
    w = v.fo[l] > w ? v.fo[l] : w;
  }
  return w;
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers (C ABI in nmq_abi.cu)

cudaError_t launch_texel_grads(const MatParams& mp, int64_t n, const float* uv, const int32_t* level,
                               const float* z_grad, float* grad, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
  const bool vec = ((uintptr_t)grad & 15u) == 0;
  // coarse tail: the last levels whose texels together fit kTailTexels
  const LevelDesc& last = mp.lv[mp.n_levels - 1];
  const int64_t total = last.off + (int64_t)last.w * last.h;
  int64_t tail_start = total;
  for (int l = mp.n_levels - 1; l >= 0 && total - mp.lv[l].off <= kTailTexels; --l) tail_start = mp.lv[l].off;
  texel_grads_kernel<<<(int)blocks, 256, 0, s>>>(mp, n, uv, level, z_grad, grad, vec, tail_start,
                                                 (int)(total - tail_start));
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_mlp_forward(const int32_t* fi, const int32_t* fo, const int32_t* act, int n_layers,
                               const float* wts, int32_t w_floats, int64_t B, const float* x,
                               float* x_cache, float* pre_cache, float* out, cudaStream_t s) {
  MlpView v{};
  v.n_layers = n_layers;
  int32_t o = 0;
  for (int l = 0; l < n_layers; ++l) {
    v.fi[l] = fi[l];
    v.fo[l] = fo[l];
    v.act[l] = act[l];
    v.w_off[l] = o;
    o += fo[l] * (fi[l] + 1);
  }
  v.w_floats = w_floats;
  const bool wide = max_width(v) > 32;  // register arrays sized to the widest layer
  const int rs = (wide ? 64 : 32) + 4;
  int32_t po = 0;
  for (int l = 0; l < n_layers; ++l) {
    v.p_off[l] = po;
    po += fo[l] * rs;
  }
  const bool pad = (size_t)po * 4 <= 200 * 1024;
  const size_t smem = (size_t)(pad ? po : w_floats) * 4;
  auto kern = wide ? (pad ? mlp_forward_kernel<64, true> : mlp_forward_kernel<64, false>)
                   : (pad ? mlp_forward_kernel<32, true> : mlp_forward_kernel<32, false>);
  const int lim = max_dynamic_smem((const void*)kern);
  if (lim < 0) return cudaErrorInvalidValue;
  if ((int)smem > lim) return cudaErrorNotSupported;  // weights larger than shared memory
  cudaError_t e;
  int64_t blocks = (B + 127) / 128;
  if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
  kern<<<(int)blocks, 128, smem, s>>>(v, B, wts, x, x_cache, pre_cache, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_mlp_backward(const int32_t* fi, const int32_t* fo, const int32_t* act, int n_layers,
                                const float* wts, int32_t w_floats, int64_t B, const float* x_cache,
                                const float* pre_cache, const float* out_grad, double* g_cache,
                                double* dparams, double* dx, cudaStream_t s) {
  MlpView v{};
  v.n_layers = n_layers;
  int32_t o = 0;
  for (int l = 0; l < n_layers; ++l) {
    v.fi[l] = fi[l];
    v.fo[l] = fo[l];
    v.act[l] = act[l];
    v.w_off[l] = o;
    o += fo[l] * (fi[l] + 1);
  }
  v.w_floats = w_floats;
  const bool wide = max_width(v) > 32, w64 = (size_t)w_floats * 8 <= 200 * 1024;
  const size_t smem = (size_t)w_floats * (w64 ? 8 : 4);  // float64 copy of the weights when it fits
  auto kern = wide ? (w64 ? mlp_backward_kernel<64, double> : mlp_backward_kernel<64, float>)
                   : (w64 ? mlp_backward_kernel<32, double> : mlp_backward_kernel<32, float>);
  const int lim = max_dynamic_smem((const void*)kern);
  if (lim < 0) return cudaErrorInvalidValue;
  if ((int)smem > lim) return cudaErrorNotSupported;  // weights larger than shared memory
  cudaError_t e;
  int64_t blocks = (B + 127) / 128;
  if (blocks > (int64_t)sm_count() * 8) blocks = (int64_t)sm_count() * 8;
  kern<<<(int)blocks, 128, smem, s>>>(v, B, wts, pre_cache, out_grad, g_cache, dx);
  ++g_launches;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(dparams, 0, (size_t)w_floats * 8, s)) != cudaSuccess) return e;
  // all layers' dW/db in one launch: the layers are independent once the
  // backward chain has cached every g, and n_layers x the CTAs hide load latency
  DparamArgs da;
  int64_t pre_off = 0;
  for (int l = 0; l < n_layers; ++l) {
    da.fi[l] = fi[l];
    da.fo[l] = fo[l];
    da.in_act[l] = l == 0 ? 0 : act[l - 1];
    da.in_src[l] = l == 0 ? x_cache : pre_cache + (pre_off - (int64_t)fo[l - 1] * B);
    da.g[l] = g_cache + pre_off;
    da.dp[l] = dparams + v.w_off[l];
    pre_off += (int64_t)fo[l] * B;
  }
#ifndef NMQ_DPARAM_TC
#define NMQ_DPARAM_TC 1  // dW / db on the tensor cores (3xTF32); 0: the float64 SIMT reduction
#endif
#ifndef NMQ_DPARAM_TMA
#define NMQ_DPARAM_TMA 1
#endif
  if (NMQ_DPARAM_TC && NMQ_DPARAM_TMA && B < ((int64_t)1 << 31) &&
      max_dynamic_smem((const void*)mlp_dparam_tma_kernel) >= (int)kTmSmem) {
    static DparamMaps maps;  // host staging of the kernel parameter (copied at launch)
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    bool ok = true;
    for (int l = 0; l < n_layers && ok; ++l) {
      ok = encode_rows(&maps.g[l], da.g[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, B, da.fo[l]) &&
           encode_rows(&maps.x[l], da.in_src[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, da.fi[l]);
    }
    if (ok) {
      int64_t rows = (B * n_layers + sm_count() - 1) / sm_count();  // ~one CTA per SM over all layers
      rows = (rows + kTmKT - 1) / kTmKT * kTmKT;
      const dim3 gt((unsigned)((B + rows - 1) / rows), (unsigned)n_layers);
      mlp_dparam_tma_kernel<<<gt, kTmThreads, kTmSmem, s>>>(da, maps, B, rows);
      ++g_launches;
      return cudaGetLastError();
    }
  }
  if (NMQ_DPARAM_TC) {
    if (max_dynamic_smem((const void*)mlp_dparam_tc_kernel) < (int)kTcSmem) return cudaErrorNotSupported;
    const dim3 gtc((unsigned)((B + kTcRows - 1) / kTcRows), (unsigned)n_layers);
    mlp_dparam_tc_kernel<<<gtc, 128, kTcSmem, s>>>(da, B);
    ++g_launches;
    return cudaGetLastError();
  }
  const dim3 grid((unsigned)((B + kRowsPerCta - 1) / kRowsPerCta), (unsigned)n_layers);
  if (wide)
    mlp_dparam_kernel<64><<<grid, 256, 0, s>>>(da, B);
  else
    mlp_dparam_kernel<32><<<grid, 256, 0, s>>>(da, B);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace nmq
