// nmq_kernels.cu — fused sm_100a kernels of the neural-material query path.
//
// Execution model:
//  * A CTA holds G "tile groups" of 128 threads.  A tile group owns one tile
//    of 128 queries at a time, one query per thread, and loops persistently
//    over tiles.  Weights of every network are staged ONCE per CTA in SMEM in
//    the UMMA K-major chunk layout (B operand).
//  * Per MLP layer a tile group writes its activations as fp16 into its
//    private TMEM region (A operand, tcgen05.st, lane = query), one elected
//    thread issues tcgen05.mma (A from TMEM, B from SMEM, D fp32 in TMEM) and
//    commits to the group's mbarrier; the threads then read D back with
//    tcgen05.ld (lane = query) and run the per-query nonlinear code.
//  * The reference keeps hidden activations in fp32 (mlp.py:205-207).  To
//    match it with fp16 tensor-core inputs every hidden activation a is
//    split a = hi + lo (hi = fp16(a), lo = fp16(a - hi)) and the layer runs
//    W*[hi; lo] with the weights duplicated along K — exact to ~2^-22.
//    Biases ride along as an extra K column against a constant 1.0.
#include <cstdio>
#include <mutex>
#include <unordered_map>
#include "tc.cuh"
#include "nmq_device.cuh"
#include "nmq_internal.h"

namespace nmq {

std::atomic<int64_t> g_launches{0};

int max_dynamic_smem(const void* kernel) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> done;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find(kernel);
  if (it != done.end()) return it->second;
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  int lim = -1;
  if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess) {
    lim = optin - (int)fa.sharedSizeBytes;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, lim) != cudaSuccess) lim = -1;
  }
  done[kernel] = lim;
  return lim;
}
int g_kernel_path = 0;
std::atomic<int> g_last_path{0};

namespace {

using namespace dev;

struct Group {
  uint32_t d0, a0;    // TMEM column of the group's D / A region (lane 0)
  uint32_t lane;      // this warp's TMEM lane field
  uint32_t bias_col;  // shared constant chunk
  uint64_t* bar;
  uint32_t phase;
  uint32_t bar_id;
  uint32_t smem_w;
  bool leader;
};

__device__ __forceinline__ uint32_t h2bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// Issue one MLP layer for the calling tile group (all 128 threads call).
__device__ __forceinline__ void run_layer(const LayerDesc& L, Group& g) {
  tc::tmem_st_wait();
  tc::tc_fence_before();
  tc::named_bar(g.bar_id, 128);
  if (g.leader) {
    tc::tc_fence_after();
    const uint32_t idesc = tc::idesc_f16(128, L.n_pad);
    const uint32_t lbo = (uint32_t)L.n_pad * 16u;
    const uint32_t b0 = g.smem_w + L.b_off;
    if (L.precise) {
      // fp32 path: A = [x_hi | x_lo] (ks k-steps each), B = [W_hi | W_hi | W_lo]:
      // W_hi x_hi + W_hi x_lo + W_lo x_hi (+ bias chunk [b_hi, 0, b_lo] vs (1, 0, 1))
      const uint32_t ks = L.first ? L.ksteps : (uint32_t)L.in_pad / 16u;
      for (uint32_t p = 0; p < 3; ++p)
        for (uint32_t s = 0; s < ks; ++s)
          tc::mma_ts(g.d0, g.a0 + 8 * (s + (p == 1 ? ks : 0)),
                     tc::smem_desc(b0 + (p * ks + s) * 2 * lbo, lbo, 128), idesc, (p | s) != 0);
      if (!L.first)
        tc::mma_ts(g.d0, g.bias_col, tc::smem_desc(b0 + 3 * ks * 2 * lbo, lbo, 128), idesc, 1);
    } else if (L.first) {
      for (uint32_t s = 0; s < L.ksteps; ++s)
        tc::mma_ts(g.d0, g.a0 + 8 * s, tc::smem_desc(b0 + s * 2 * lbo, lbo, 128), idesc, s > 0);
    } else {
      const uint32_t nhl = 2u * (L.in_pad / 16u);
      for (uint32_t s = 0; s < nhl; ++s)
        tc::mma_ts(g.d0, g.a0 + 8 * s, tc::smem_desc(b0 + s * 2 * lbo, lbo, 128), idesc, s > 0);
      tc::mma_ts(g.d0, g.bias_col, tc::smem_desc(b0 + nhl * 2 * lbo, lbo, 128), idesc, 1);
    }
    tc::mma_commit(g.bar);
  }
  tc::mbar_wait(g.bar, g.phase);
  g.phase ^= 1u;
  tc::tc_fence_after();
}

// First-layer input: x[0..2*NC) as fp16 pairs into A columns [0, NC)
// (fp16 path: the input rounded to fp16 once, mlp.py:205); with `precise`
// the fp32 input as hi pairs in [0, NC) and lo pairs in [NC, 2 NC).
template <int NC>
__device__ __forceinline__ void write_input(const Group& g, const float* x, bool precise = false) {
  uint32_t r[NC];
  if (precise) {
    uint32_t lo[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const __half2 h = __floats2half2_rn(x[2 * j], x[2 * j + 1]);
      const float2 hf = __half22float2(h);
      r[j] = h2bits(h);
      lo[j] = h2bits(__floats2half2_rn(x[2 * j] - hf.x, x[2 * j + 1] - hf.y));
    }
#pragma unroll
    for (int c = 0; c < NC; c += 8) {
      uint32_t q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = lo[c + j];
      tc::tmem_st8(g.lane + g.a0 + NC + c, q);
    }
  } else {
#pragma unroll
    for (int j = 0; j < NC; ++j) r[j] = h2bits(__floats2half2_rn(x[2 * j], x[2 * j + 1]));
  }
  if constexpr (NC == 8) {
    tc::tmem_st8(g.lane + g.a0, r);
  } else {
#pragma unroll
    for (int c = 0; c < NC; c += 8) {
      uint32_t q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = r[c + j];
      tc::tmem_st8(g.lane + g.a0 + c, q);
    }
  }
}

// Hidden epilogue: D[0, width) -> act -> (hi, lo) fp16 into A.
__device__ __forceinline__ void hidden_epilogue(const Group& g, uint32_t width, bool leaky) {
  const uint32_t half_w = width / 2;
  for (uint32_t c0 = 0; c0 < width; c0 += 16) {
    uint32_t r[16];
    tc::tmem_ld16(g.lane + g.d0 + c0, r);
    tc::tmem_ld_wait();
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float a = __uint_as_float(r[2 * j]), b = __uint_as_float(r[2 * j + 1]);
      if (leaky) {
        a = fmaxf(a, kLeaky * a);
        b = fmaxf(b, kLeaky * b);
      }
      const __half2 h = __floats2half2_rn(a, b);
      const float2 hf = __half22float2(h);
      hi[j] = h2bits(h);
      lo[j] = h2bits(__floats2half2_rn(a - hf.x, b - hf.y));
    }
    tc::tmem_st8(g.lane + g.a0 + c0 / 2, hi);
    tc::tmem_st8(g.lane + g.a0 + half_w + c0 / 2, lo);
  }
}

// Output layer: first 16 columns of D
__device__ __forceinline__ void output_epilogue(const Group& g, float (&y)[16]) {
  uint32_t r[16];
  tc::tmem_ld16(g.lane + g.d0, r);
  tc::tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 16; ++j) y[j] = __uint_as_float(r[j]);
}

// Run a chain of layers [first, first+count) whose first layer input is
// already in A.  Leaves the last layer's raw outputs in y.
__device__ __forceinline__ void run_chain(const MatParams& mp, int first, int count, Group& g,
                                          float (&y)[16]) {
  run_layer(mp.layers[first], g);
  for (int i = 1; i < count; ++i) {
    const LayerDesc& prev = mp.layers[first + i - 1];
    hidden_epilogue(g, prev.n_pad, prev.act != 0);
    run_layer(mp.layers[first + i], g);
  }
  output_epilogue(g, y);
}

__device__ __forceinline__ void load_z(const float* z, int64_t q, float (&out)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(z + 8 * q));
  const float4 b = __ldg(reinterpret_cast<const float4*>(z + 8 * q + 4));
  out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
  out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
}

// BRDF decode of one query given z; returns raw decoder outputs in y.
// wi64 / wo64: the query's float64 directions when the caller passed them,
// else null — the reference transforms its float64 arrays.
// PREC: instantiated for precise (fp32-master) materials only — the fp16
// path's reference-arithmetic frames (IEEE divisions with slow-path calls)
// are compiled out of it (their register pressure measured -7 % there).
template <bool PREC = false>
__device__ __forceinline__ void brdf_decode(const MatParams& mp, Group& g, const float (&z)[8],
                                            V3 wi, V3 wo, float (&y)[16], const double* wi64 = nullptr,
                                            const double* wo64 = nullptr) {
  float x[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = z[k];
  if (!PREC && mp.use_frames && !mp.precise) {
    // fp16 path: the reference's rounding of every decoder input, exactly —
    // frame layer in its sequential-FMA order, frames and transforms in
    // float64, fp32, then fp16 (neural.py:282-287)
    uint32_t zh[4], x16[6];
#pragma unroll
    for (int c = 0; c < 4; ++c) zh[c] = pack_h2(z[2 * c], z[2 * c + 1]);
    // float64 directions are read here, at the point of use (nothing float64
    // stays live across the fetch); one call site keeps the code single
    const D3 di = wi64 ? D3{__ldg(wi64), __ldg(wi64 + 1), __ldg(wi64 + 2)} : d3(wi);
    const D3 dq = wo64 ? D3{__ldg(wo64), __ldg(wo64 + 1), __ldg(wo64 + 2)} : d3(wo);
    tw_exact(mp, zh, di, dq, x16);
#pragma unroll
    for (int c = 0; c < 6; ++c) {
      const float2 f = unpack_h2(x16[c]);
      x[8 + 2 * c] = f.x;
      x[9 + 2 * c] = f.y;
    }
  } else if (mp.use_frames) {
    float xf[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) xf[k] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) xf[k] = z[k];
    xf[8] = 1.f;  // bias slot
    write_input<8>(g, xf, mp.precise != 0);
    run_layer(mp.layers[mp.frame_layer], g);
    float raw[16];
    output_epilogue(g, raw);
    // frames_from_raw + transform (neural.py:207-233, 185-196, 284-286):
    // decoder input [z, T1 wi, T2 wi, T1 wo, T2 wo] (tests/test_neural.py:105-118)
    float ti[6], to[6];
#pragma unroll
    for (int f = 0; f < 2; ++f) {
      const Frame fr = frame_from_raw(raw + 6 * f);
      ti[3 * f + 0] = dot(fr.t, wi);
      ti[3 * f + 1] = dot(fr.b, wi);
      ti[3 * f + 2] = dot(fr.n, wi);
      to[3 * f + 0] = dot(fr.t, wo);
      to[3 * f + 1] = dot(fr.b, wo);
      to[3 * f + 2] = dot(fr.n, wo);
    }
    if (mp.n_frames == 2) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        x[8 + k] = ti[k];
        x[14 + k] = to[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        x[8 + k] = ti[k];
        x[11 + k] = to[k];
      }
    }
  } else {
    x[8] = wi.x; x[9] = wi.y; x[10] = wi.z;
    x[11] = wo.x; x[12] = wo.y; x[13] = wo.z;
  }
  // bias slot of the first BRDF layer (index = fan_in)
  if (mp.brdf_in == 20) x[20] = 1.f;  // 2 frames
  else x[14] = 1.f;                   // 1 frame or no frames (host-validated)
  if (mp.layers[mp.brdf_first].ksteps == 1) write_input<8>(g, x, mp.precise != 0);
  else write_input<16>(g, x, mp.precise != 0);
  run_chain(mp, mp.brdf_first, mp.brdf_count, g, y);
}

__device__ __forceinline__ Proxy sampler_decode(const MatParams& mp, Group& g,
                                                const float (&z)[8], V3 wi) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = z[k];
  x[8] = wi.x; x[9] = wi.y; x[10] = wi.z;
  x[11] = 1.f;  // bias slot
#pragma unroll
  for (int k = 12; k < 16; ++k) x[k] = 0.f;
  write_input<8>(g, x, mp.precise != 0);
  float y[16];
  run_chain(mp, mp.samp_first, mp.samp_count, g, y);
  return proxy_from_raw(y, mp.isotropic != 0);
}

template <int MODE, bool PREC>
__global__ void __launch_bounds__(384, 2)
fused_kernel(const __grid_constant__ MatParams mp, const __grid_constant__ QueryArgs a,
             uint32_t tmem_cols, uint32_t group_cols) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tbase_sh;
  const int tid = threadIdx.x;
  const int G = blockDim.x / 128;
  const int gi = tid / 128, r = tid % 128;
  const int warp = tid / 32;

  // --- one-time CTA setup: weights -> SMEM, barriers, TMEM -----------------
  {
    const uint4* src = mp.wblob;
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = mp.wblob_bytes / 16;
    for (uint32_t i = tid; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  if (tid < G) tc::mbar_init(&bars[tid], 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tbase_sh)), "r"(tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_proxy_async_smem();
  tc::fence_mbar_init();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase_sh;
  const uint32_t bias_col = tb + (uint32_t)G * group_cols;
  if (warp < 4) {
    const uint32_t v[8] = {0x3C00u, 0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u};  // fp16 1.0 at k = 0, 2
    tc::tmem_st8(bias_col + ((uint32_t)(warp * 32) << 16), v);
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  Group g;
  g.d0 = tb + (uint32_t)gi * group_cols;
  g.a0 = g.d0 + group_cols / 2;
  g.lane = (uint32_t)((warp & 3) * 32) << 16;
  g.bias_col = bias_col;
  g.bar = &bars[gi];
  g.phase = 0;
  g.bar_id = 1 + gi;
  g.smem_w = tc::smem_u32(smem);
  g.leader = (r == 0);

  const int64_t seg_base = a.seg ? (int64_t)__ldg(a.seg) : 0;  // binned segment rows
  const int64_t n_rows = a.seg ? (int64_t)__ldg(a.seg + 1) : a.n;
  const int64_t ntiles = (n_rows + kTile - 1) / kTile;
  for (int64_t tile = (int64_t)blockIdx.x * G + gi; tile < ntiles;
       tile += (int64_t)gridDim.x * G) {
    const int64_t i = tile * kTile + r;
    const bool valid = i < n_rows;
    const int64_t q = valid ? (a.idx ? (int64_t)__ldg(a.idx + seg_base + i) : seg_base + i) : 0;
    const int64_t oq = valid ? (a.out_idx ? (int64_t)__ldg(a.out_idx + seg_base + i) : q) : 0;  // output row

    V3 wi = v3(0.f, 0.f, 1.f), wo = v3(0.f, 0.f, 1.f);
    auto load_dirs = [&](bool with_wo) {
      if (a.wi64) {  // narrowed copies for the fp32 consumers (sampler input, proxy)
        wi = v3((float)__ldg(a.wi64 + 3 * q), (float)__ldg(a.wi64 + 3 * q + 1), (float)__ldg(a.wi64 + 3 * q + 2));
        if (with_wo)
          wo = v3((float)__ldg(a.wo64 + 3 * q), (float)__ldg(a.wo64 + 3 * q + 1), (float)__ldg(a.wo64 + 3 * q + 2));
      } else {
        wi = ldg3(a.wi, q);
        if (with_wo) wo = ldg3(a.wo, q);
      }
    };
    float z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = 0.f;

    if constexpr (MODE == kModeEvalZ || MODE == kModeProxyZ) {
      if (valid) {
        load_z(a.z, q, z);
        load_dirs(MODE == kModeEvalZ);
      }
    } else {
      if (a.uv64) {  // float64 coordinates, as the reference computes them
        double u = 0.0, v = 0.0, lod = 0.0, urr = 0.0;
        if (valid) {
          u = __ldg(a.uv64 + 2 * q);
          v = __ldg(a.uv64 + 2 * q + 1);
          lod = __ldg(a.lod64 + (a.lod_stride ? q : 0));
          urr = __ldg(a.urr64 + q);
          load_dirs(MODE != kModeSamplePdf);
        }
        const int level = choose_level(mp, lod, urr);
        fetch_exact(mp, level, u, v, make_taps(mp, level, u, v), z);
        if (valid && a.level) a.level[oq] = level;
      } else {
        float u = 0.f, v = 0.f, lod = 0.f, urr = 0.f;
        if (valid) {
          const float2 uv = __ldg(reinterpret_cast<const float2*>(a.uv) + q);
          u = uv.x;
          v = uv.y;
          lod = __ldg(a.lod + (a.lod_stride ? q : 0));
          urr = __ldg(a.u_rr + q);
          load_dirs(MODE != kModeSamplePdf);
        }
        const int level = choose_level(mp, lod, urr);
        const Taps t = make_taps(mp, level, u, v);
        fetch_exact(mp, level, u, v, t, z);
        if (valid && a.level) a.level[oq] = level;
      }
    }

    if constexpr (MODE == kModeEval || MODE == kModeEvalZ || MODE == kModeQuery) {
      float y[16];
      const bool d64 = a.wi64 && valid;
      brdf_decode<PREC>(mp, g, z, wi, wo, y, d64 ? a.wi64 + 3 * q : nullptr, d64 ? a.wo64 + 3 * q : nullptr);
      // horizon mask on the caller's values (a float64 z below 2^-149 narrows to 0)
      const bool up = d64 ? (__ldg(a.wi64 + 3 * q + 2) > 0.0 && __ldg(a.wo64 + 3 * q + 2) > 0.0)
                          : (wi.z > 0.f && wo.z > 0.f);
      if (MODE == kModeEval && a.img) {  // per-pixel spp mean (warp-collective)
        const V3 f = up ? v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2])) : v3(0.f, 0.f, 0.f);
        spp_accumulate(a.img, i, f, valid, a.spp_log2);
      } else if (valid) {
        const V3 f = up ? v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2]))
                        : v3(0.f, 0.f, 0.f);
        stg3(a.rgb, oq, f);
        if (mp.albedo && a.albedo) {
          const V3 al = up ? v3(fmaxf(y[3], 0.f), fmaxf(y[4], 0.f), fmaxf(y[5], 0.f))
                           : v3(0.f, 0.f, 0.f);
          stg3(a.albedo, oq, al);
        }
      }
    }
    if constexpr (MODE == kModeProxyZ || MODE == kModeSamplePdf || MODE == kModeQuery) {
      const Proxy p = sampler_decode(mp, g, z, wi);
      if (valid) {
        if (a.params9) store_proxy(a.params9, oq, p);
        if constexpr (MODE != kModeProxyZ) {
          const V3 u3 = ldg3(a.u3, q);
          const V3 s = proxy_sample(p, wi, u3.x, u3.y, u3.z);
          stg3(a.ws, oq, s);
          a.pdf[oq] = proxy_pdf(p, wi, s);
        }
      }
    }
  }

  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(tmem_cols)
                 : "memory");
  }
}

// --- DIVERGENT multi-material eval --------------------------------------------
// Every material's parameter block and weights live in SMEM.  Each thread
// fetches its latent code from its own material's pyramid; the tile then
// loops over the materials present in it (warp ballots OR-ed across the
// tile group) and decodes all 128 rows with each, keeping its own.
__global__ void __launch_bounds__(384, 1)
divergent_eval_kernel(const MatParams* __restrict__ mps_g, int32_t n_mats,
                      const __grid_constant__ QueryArgs a, const int32_t* __restrict__ mat_id,
                      uint32_t tmem_cols, uint32_t group_cols) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tbase_sh;
  __shared__ uint32_t mask_sh[8];
  __shared__ uint32_t boff_sh[32];
  const int tid = threadIdx.x;
  const int G = blockDim.x / 128;
  const int gi = tid / 128, r = tid % 128;
  const int warp = tid / 32;

  MatParams* mps = reinterpret_cast<MatParams*>(smem);
  {
    const uint4* src = reinterpret_cast<const uint4*>(mps_g);
    uint4* dst = reinterpret_cast<uint4*>(smem);
    const uint32_t n16 = (uint32_t)(n_mats * sizeof(MatParams) / 16);
    for (uint32_t i = tid; i < n16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t off = ((uint32_t)(n_mats * sizeof(MatParams)) + 127u) & ~127u;
    for (int k = 0; k < n_mats; ++k) {
      boff_sh[k] = off;
      off += (mps[k].wblob_bytes + 127u) & ~127u;
    }
  }
  __syncthreads();
  for (int k = 0; k < n_mats; ++k) {
    const uint4* src = mps[k].wblob;
    uint4* dst = reinterpret_cast<uint4*>(smem + boff_sh[k]);
    for (uint32_t i = tid; i < mps[k].wblob_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  if (tid < G) tc::mbar_init(&bars[tid], 1);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     tc::smem_u32(&tbase_sh)), "r"(tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc::fence_proxy_async_smem();
  tc::fence_mbar_init();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase_sh;
  const uint32_t bias_col = tb + (uint32_t)G * group_cols;
  if (warp < 4) {
    const uint32_t v[8] = {0x3C00u, 0x3C00u, 0u, 0u, 0u, 0u, 0u, 0u};
    tc::tmem_st8(bias_col + ((uint32_t)(warp * 32) << 16), v);
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  Group g;
  g.d0 = tb + (uint32_t)gi * group_cols;
  g.a0 = g.d0 + group_cols / 2;
  g.lane = (uint32_t)((warp & 3) * 32) << 16;
  g.bias_col = bias_col;
  g.bar = &bars[gi];
  g.phase = 0;
  g.bar_id = 1 + gi;
  g.leader = (r == 0);
  const uint32_t smem_base = tc::smem_u32(smem);

  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  for (int64_t tile = (int64_t)blockIdx.x * G + gi; tile < ntiles;
       tile += (int64_t)gridDim.x * G) {
    const int64_t q = tile * kTile + r;
    const int m0 = q < a.n ? __ldg(mat_id + q) : -1;
    const bool valid = m0 >= 0 && m0 < n_mats;  // out-of-range ids are skipped
    const int m = valid ? m0 : -1;
    V3 wi = v3(0.f, 0.f, 1.f), wo = v3(0.f, 0.f, 1.f);
    auto load_dirs = [&](bool with_wo) {
      if (a.wi64) {  // narrowed copies for the fp32 consumers (sampler input, proxy)
        wi = v3((float)__ldg(a.wi64 + 3 * q), (float)__ldg(a.wi64 + 3 * q + 1), (float)__ldg(a.wi64 + 3 * q + 2));
        if (with_wo)
          wo = v3((float)__ldg(a.wo64 + 3 * q), (float)__ldg(a.wo64 + 3 * q + 1), (float)__ldg(a.wo64 + 3 * q + 2));
      } else {
        wi = ldg3(a.wi, q);
        if (with_wo) wo = ldg3(a.wo, q);
      }
    };
    float z[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = 0.f;
    if (valid) {
      const MatParams& mm = mps[m];
      const float2 uv = __ldg(reinterpret_cast<const float2*>(a.uv) + q);
      const float lod = __ldg(a.lod + (a.lod_stride ? q : 0));
      const int level = choose_level(mm, lod, __ldg(a.u_rr + q));
      const Taps t = make_taps(mm, level, uv.x, uv.y);
      fetch_exact(mm, level, uv.x, uv.y, t, z);
      wi = ldg3(a.wi, q);
      wo = ldg3(a.wo, q);
      if (a.level) a.level[q] = level;
    }
    // materials present in this tile
    const uint32_t wmask = __reduce_or_sync(0xffffffffu, valid ? (1u << m) : 0u);
    if (r == 0) mask_sh[gi] = 0u;
    tc::named_bar(g.bar_id, 128);
    if ((r & 31) == 0) atomicOr(&mask_sh[gi], wmask);
    tc::named_bar(g.bar_id, 128);
    uint32_t mask = mask_sh[gi];
    float y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) y[j] = 0.f;
    while (mask) {
      const int k = __ffs(mask) - 1;
      mask &= mask - 1;
      g.smem_w = smem_base + boff_sh[k];
      float yk[16];
      brdf_decode(mps[k], g, z, wi, wo, yk);
      if (m == k) {
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = yk[j];
      }
    }
    if (valid) {
      const bool up = (wi.z > 0.f) && (wo.z > 0.f);
      const V3 f = up ? v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2]))
                      : v3(0.f, 0.f, 0.f);
      stg3(a.rgb, q, f);
    }
  }

  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(tmem_cols)
                 : "memory");
  }
}

// --- plain SIMT kernels ------------------------------------------------------
__global__ void __launch_bounds__(256) fetch_kernel(const __grid_constant__ MatParams mp,
                                                    const __grid_constant__ QueryArgs a) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (a.uv64) {  // float64 coordinates
      const double u = __ldg(a.uv64 + 2 * i), v = __ldg(a.uv64 + 2 * i + 1);
      const int level = choose_level(mp, __ldg(a.lod64 + (a.lod_stride ? i : 0)), __ldg(a.urr64 + i));
      const Taps t = make_taps(mp, level, u, v);
      float z[8];
      fetch_exact(mp, level, u, v, t, z);
      if (a.z_out) {
        float4* o = reinterpret_cast<float4*>(a.z_out + 8 * i);
        o[0] = make_float4(z[0], z[1], z[2], z[3]);
        o[1] = make_float4(z[4], z[5], z[6], z[7]);
      }
      if (a.level) a.level[i] = level;
      if (a.taps) {
        int32_t* p = a.taps + 8 * i;
        p[0] = t.x0; p[1] = t.y0; p[2] = t.x1; p[3] = t.y0;
        p[4] = t.x0; p[5] = t.y1; p[6] = t.x1; p[7] = t.y1;
      }
      if (a.wts) {
        double w[4];
        weights64(frac64d(u, mp.lv[level].w), frac64d(v, mp.lv[level].h), w);
        float* o = a.wts + 4 * i;
        o[0] = (float)w[0]; o[1] = (float)w[1]; o[2] = (float)w[2]; o[3] = (float)w[3];
      }
      continue;
    }
    const float2 uv = __ldg(reinterpret_cast<const float2*>(a.uv) + i);
    const float lod = __ldg(a.lod + (a.lod_stride ? i : 0));
    if (a.trilinear) {
      // (1 - f) * bilinear(floor l) + f * bilinear(ceil l) in float64 from the
      // two float32 fetches (the roulette's expectation, latent.py:84-92)
      const float top = (float)(mp.n_levels - 1);
      const float l = fminf(fmaxf(lod, 0.f), top);
      const int lo = (int)floorf(l), hi = lo + 1 < mp.n_levels ? lo + 1 : lo;
      const double f = (double)l - (double)floorf(l);
      float za[8], zb[8];
      fetch_exact(mp, lo, uv.x, uv.y, make_taps(mp, lo, uv.x, uv.y), za);
      fetch_exact(mp, hi, uv.x, uv.y, make_taps(mp, hi, uv.x, uv.y), zb);
      float z[8];
#pragma unroll
      for (int c = 0; c < 8; ++c)
        z[c] = (float)__dadd_rn(__dmul_rn(__dsub_rn(1.0, f), (double)za[c]), __dmul_rn(f, (double)zb[c]));
      float4* o = reinterpret_cast<float4*>(a.z_out + 8 * i);
      o[0] = make_float4(z[0], z[1], z[2], z[3]);
      o[1] = make_float4(z[4], z[5], z[6], z[7]);
      if (a.level) a.level[i] = lo;
      continue;
    }
    const int level = choose_level(mp, lod, __ldg(a.u_rr + i));
    const Taps t = make_taps(mp, level, uv.x, uv.y);
    float z[8];
    fetch_exact(mp, level, uv.x, uv.y, t, z);
    if (a.z_out) {
      float4* o = reinterpret_cast<float4*>(a.z_out + 8 * i);
      o[0] = make_float4(z[0], z[1], z[2], z[3]);
      o[1] = make_float4(z[4], z[5], z[6], z[7]);
    }
    if (a.level) a.level[i] = level;
    if (a.taps) {
      int32_t* p = a.taps + 8 * i;
      p[0] = t.x0; p[1] = t.y0; p[2] = t.x1; p[3] = t.y0;
      p[4] = t.x0; p[5] = t.y1; p[6] = t.x1; p[7] = t.y1;
    }
    if (a.wts) {
      double w[4];
      weights64(frac64(uv.x, mp.lv[level].w), frac64(uv.y, mp.lv[level].h), w);
      float* o = a.wts + 4 * i;
      o[0] = (float)w[0]; o[1] = (float)w[1]; o[2] = (float)w[2]; o[3] = (float)w[3];
    }
  }
}

__global__ void __launch_bounds__(256) sample_kernel(int64_t n, const float* __restrict__ p9,
                                                     const float* __restrict__ wi,
                                                     const float* __restrict__ u3,
                                                     float* __restrict__ wo) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const Proxy p = load_proxy(p9, i);
    const V3 u = ldg3(u3, i);
    stg3(wo, i, proxy_sample(p, ldg3(wi, i), u.x, u.y, u.z));
  }
}

__global__ void __launch_bounds__(256) pdf_kernel(int64_t n, const float* __restrict__ p9,
                                                  const float* __restrict__ wi,
                                                  const float* __restrict__ wo,
                                                  float* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = proxy_pdf(load_proxy(p9, i), ldg3(wi, i), ldg3(wo, i));
  }
}

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

int grid_for(int64_t n, int block) {
  int64_t blocks = (n + block - 1) / block;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

template <int MODE>
cudaError_t launch_mode(const MatParams& mp, const QueryArgs& a, cudaStream_t s, int groups) {
  const uint32_t group_cols = 2u * (uint32_t)mp.dmax;
  // tile groups per CTA; TMEM budget = G*group_cols + 8 (bias chunk), pow2
  int G = groups > 0 ? groups : (mp.dmax <= 32 ? 3 : 3);
  if (G > 3) G = 3;  // __launch_bounds__(384)
  uint32_t need = (uint32_t)G * group_cols + 8u;
  uint32_t cols = 32;
  while (cols < need) cols <<= 1;
  if (cols > 512) return cudaErrorInvalidValue;
  const int ctas_per_sm = (int)(512 / cols) < 2 ? (int)(512 / cols) : 2;
  const int smem = smem_bytes_for(mp);
  auto kern = mp.precise ? fused_kernel<MODE, true> : fused_kernel<MODE, false>;
  const int lim = max_dynamic_smem((const void*)kern);
  if (lim < 0) return cudaErrorInvalidValue;
  if (smem > lim) return cudaErrorNotSupported;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  int64_t grid = (int64_t)num_sms() * ctas_per_sm;
  if (a.max_ctas > 0 && grid > (int64_t)a.max_ctas * ctas_per_sm) grid = (int64_t)a.max_ctas * ctas_per_sm;
  const int64_t need_ctas = (ntiles + G - 1) / G;
  if (grid > need_ctas) grid = need_ctas;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, G * 128, smem, s>>>(mp, a, cols, group_cols);
  ++g_launches;
  return cudaGetLastError();
}

// The decoder's fp16 direction inputs, one row per thread, in the
// reference's arithmetic (the check hook behind nm_decoder_inputs).
__global__ void __launch_bounds__(256) decoder_inputs_kernel(const __grid_constant__ MatParams mp, int64_t n,
                                                             const float* __restrict__ z,
                                                             const float* __restrict__ wi,
                                                             const float* __restrict__ wo,
                                                             const double* __restrict__ wi64,
                                                             const double* __restrict__ wo64,
                                                             uint32_t* __restrict__ x16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float zz[8];
    load_z(z, i, zz);
    uint32_t zh[4], x[6];
#pragma unroll
    for (int c = 0; c < 4; ++c) zh[c] = pack_h2(zz[2 * c], zz[2 * c + 1]);
    if (wi64)
      tw_exact(mp, zh, D3{wi64[3 * i], wi64[3 * i + 1], wi64[3 * i + 2]},
               D3{wo64[3 * i], wo64[3 * i + 1], wo64[3 * i + 2]}, x);
    else
      tw_exact(mp, zh, ldg3(wi, i), ldg3(wo, i), x);
#pragma unroll
    for (int c = 0; c < 6; ++c) x16[6 * i + c] = x[c];
  }
}

}  // namespace

int smem_bytes_for(const MatParams& mp) { return (int)((mp.wblob_bytes + 127) / 128 * 128); }

cudaError_t launch_fused(const MatParams& mp, int mode, const QueryArgs& a, cudaStream_t s,
                         int groups) {
  if (a.n <= 0) return cudaSuccess;
  if (groups == 0 && (g_kernel_path == 0 || g_kernel_path == 2)) {
    const cudaError_t e = launch_fast(mp, mode, a, s);
    if (e != cudaErrorNotSupported) return g_last_path.store(2), e;
    (void)cudaGetLastError();
  }
  g_last_path = 1;
  switch (mode) {
    case kModeEval: return launch_mode<kModeEval>(mp, a, s, groups);
    case kModeEvalZ: return launch_mode<kModeEvalZ>(mp, a, s, groups);
    case kModeProxyZ: return launch_mode<kModeProxyZ>(mp, a, s, groups);
    case kModeSamplePdf: return launch_mode<kModeSamplePdf>(mp, a, s, groups);
    case kModeQuery: return launch_mode<kModeQuery>(mp, a, s, groups);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_eval_divergent(const MatParams* const* mps_host, const MatParams* mps_dev,
                                  int32_t n_mats, const int32_t* mat_id, const QueryArgs& a,
                                  cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  uint32_t smem = ((uint32_t)(n_mats * sizeof(MatParams)) + 127u) & ~127u;
  int dmax = 16;
  for (int k = 0; k < n_mats; ++k) {
    smem += (mps_host[k]->wblob_bytes + 127u) & ~127u;
    dmax = dmax > mps_host[k]->dmax ? dmax : mps_host[k]->dmax;
  }
  if (smem > 220u * 1024u) return cudaErrorInvalidValue;
  const uint32_t group_cols = 2u * (uint32_t)dmax;
  const int G = 3;
  uint32_t need = G * group_cols + 8u, cols = 32;
  while (cols < need) cols <<= 1;
  if (cols > 512) return cudaErrorInvalidValue;
  const int lim = max_dynamic_smem((const void*)divergent_eval_kernel);
  if (lim < 0 || (int)smem > lim) return cudaErrorInvalidValue;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  int64_t grid = num_sms();
  if (grid > (ntiles + G - 1) / G) grid = (ntiles + G - 1) / G;
  divergent_eval_kernel<<<(int)grid, G * 128, smem, s>>>(mps_dev, n_mats, a, mat_id, cols,
                                                          group_cols);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_fetch(const MatParams& mp, const QueryArgs& a, cudaStream_t s) {
  if (a.n <= 0) return cudaSuccess;
  fetch_kernel<<<grid_for(a.n, 256), 256, 0, s>>>(mp, a);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_sample(int64_t n, const float* p9, const float* wi, const float* u3, float* wo,
                          cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  sample_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, p9, wi, u3, wo);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_pdf(int64_t n, const float* p9, const float* wi, const float* wo, float* pdf,
                       cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pdf_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, p9, wi, wo, pdf);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_decoder_inputs(const MatParams& mp, int64_t n, const float* z, const float* wi,
                                  const float* wo, const double* wi64, const double* wo64, uint32_t* x16,
                                  cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  decoder_inputs_kernel<<<(unsigned)blocks, 256, 0, s>>>(mp, n, z, wi, wo, wi64, wo64, x16);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace nmq
