// nmq_fast.cu — pipelined, architecture-specialized fused query kernels
// (the coherent per-material path).
//
// One persistent CTA per SM holds G tile groups of 128 threads; each group
// loops over 128-query tiles with a three-stage software pipeline:
//
//   iteration i (tile t, next tiles t1 = t+s, t2 = t+2s):
//     (a) read tile t's inputs from SMEM (TMA'd there one iteration ago)
//     (b) blend tile t's texels (cp.async'd into SMEM one iteration ago)
//     (c) tile t1: wait its TMA'd inputs, choose level + taps, issue the
//         4 texel gathers (cp.async, 16 B each) into SMEM
//     (d) MLP chains of tile t on the tensor cores (tcgen05.mma, A and D in
//         TMEM, weights in SMEM); right after the first layer's barrier the
//         leader issues tile t2's input TMA bulk copies
//     (e) nonlinear heads + stores of tile t
//
// so HBM latency of inputs and texel gathers hides behind the previous
// tile's MLP chain.  Hidden activations use the scaled-leaky trick:
//     a~ = y + k|y|  (k = 99/101)  =  c * leaky(y),  c = 1 + k
// (one FFMA with an |.| operand modifier instead of FMUL+FMNMX); the scale
// propagates through the (positively homogeneous) network and is undone on
// the raw outputs; layer biases are multiplied by c^depth inside the MMA via
// an fp16 (hi, lo) pair in the TMEM bias chunk.  The hi/lo split itself is
// F2FP (pack) + FHFMA (a - f32(hi), mixed-precision FMA) + F2FP.
#include <cstdio>
#include <cmath>
#include "tc.cuh"
#include "nmq_device.cuh"
#include "nmq_internal.h"

namespace nmq {
namespace {

using namespace dev;

constexpr float kLk = 0.98019802570343017578f;  // fp32(99/101)

struct FastConsts {
  uint32_t beta[4];  // fp16 (hi | lo << 16) of c^j
  float inv_brdf;    // 1 / c^(brdf leaky layers)
  float inv_samp;    // 1 / c^(sampler leaky layers)
};

// per-group SMEM staging
struct InBuf {
  float uv[2 * kTile];
  float lod[kTile];
  float urr[kTile];
  float wi[3 * kTile];
  float wo[3 * kTile];
  float u3[3 * kTile];
};
struct GroupSmem {
  InBuf in[2];
  float4 aux[kTile];     // fx, fy, level bits, -
  uint4 tex[4 * kTile];  // [tap][row]
};

struct FG {
  uint32_t dl, al;  // TMEM addresses with this warp's lane field (ld/st)
  uint32_t d0, a0;  // lane-0 TMEM addresses (MMA operands)
  uint32_t bias0;   // bias chunk j at bias0 + 8j
  uint64_t* bar;
  uint32_t ph;
  uint32_t bar_id;
  uint32_t wsm;
  bool leader;
};

__device__ __forceinline__ void split_scaled(uint32_t ra, uint32_t rb, uint32_t& hi, uint32_t& lo) {
  // a~ = y + k|y|, then (hi, lo) fp16 with hi + lo = a~ to ~2^-22
  const float a = fmaf(fabsf(__uint_as_float(ra)), kLk, __uint_as_float(ra));
  const float b = fmaf(fabsf(__uint_as_float(rb)), kLk, __uint_as_float(rb));
  asm("{\n\t.reg .f16 h0, h1, m1;\n\t.reg .f32 r0, r1;\n\t"
      "cvt.rn.satfinite.f16x2.f32 %0, %3, %2;\n\t"
      "mov.b32 {h0, h1}, %0;\n\t"
      "mov.b16 m1, 0xBC00;\n\t"
      "fma.rn.f32.f16 r0, h0, m1, %2;\n\t"
      "fma.rn.f32.f16 r1, h1, m1, %3;\n\t"
      "cvt.rn.f16x2.f32 %1, r1, r0;\n\t}"
      : "=r"(hi), "=r"(lo)
      : "f"(a), "f"(b));
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// One MMA layer: KA k-steps against A in TMEM (+ the bias chunk when HID).
// `after_issue` runs on the leader right after the MMAs are issued (used to
// launch the next input TMA once every thread has passed the barrier).
template <int N, int KA, bool HID, class F>
__device__ __forceinline__ void mma_layer(FG& g, uint32_t b_off, int bias_chunk, F&& after_issue) {
  tc::tmem_st_wait();
  tc::tc_fence_before();
  tc::named_bar(g.bar_id, 128);
  if (g.leader) {
    tc::tc_fence_after();
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    constexpr uint32_t lbo = N * 16;
    const uint32_t b0 = g.wsm + b_off;
#pragma unroll
    for (int s = 0; s < KA; ++s)
      tc::mma_ts(g.d0, g.a0 + 8 * s, tc::smem_desc(b0 + s * 2 * lbo, lbo, 128), idesc, s > 0);
    if constexpr (HID)
      tc::mma_ts(g.d0, g.bias0 + 8 * bias_chunk, tc::smem_desc(b0 + KA * 2 * lbo, lbo, 128), idesc,
                 1);
    tc::mma_commit(g.bar);
    after_issue();
  }
  tc::mbar_wait(g.bar, g.ph);
  g.ph ^= 1u;
  tc::tc_fence_after();
}
struct NoOp {
  __device__ void operator()() const {}
};

// D[0, W) -> scaled leaky -> (hi, lo) into A
template <int W>
__device__ __forceinline__ void hidden_epi(const FG& g) {
  if constexpr (W == 16) {
    uint32_t r[16];
    tc::tmem_ld16(g.dl, r);
    tc::tmem_ld_wait();
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) split_scaled(r[2 * j], r[2 * j + 1], hi[j], lo[j]);
    tc::tmem_st8(g.al, hi);
    tc::tmem_st8(g.al + 8, lo);
  } else {
#pragma unroll
    for (int c0 = 0; c0 < W; c0 += 32) {
      uint32_t r[32];
      tc::tmem_ld32(g.dl + c0, r);
      tc::tmem_ld_wait();
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) split_scaled(r[2 * j], r[2 * j + 1], hi[j], lo[j]);
      tc::tmem_st16(g.al + c0 / 2, hi);
      tc::tmem_st16(g.al + W / 2 + c0 / 2, lo);
    }
  }
}

// chain: first layer (input already in A) + (NH-1) hidden + output (N=16)
template <int W, int NH, int KA0, class F>
__device__ __forceinline__ void run_chain(FG& g, const MatParams& mp, int first, F&& after_first,
                                          uint32_t (&y)[16]) {
  mma_layer<W, KA0, false>(g, mp.layers[first].b_off, 0, after_first);
#pragma unroll
  for (int i = 1; i < NH; ++i) {
    hidden_epi<W>(g);
    mma_layer<W, 2 * W / 16, true>(g, mp.layers[first + i].b_off, i, NoOp{});
  }
  hidden_epi<W>(g);
  mma_layer<16, 2 * W / 16, true>(g, mp.layers[first + NH].b_off, NH, NoOp{});
  tc::tmem_ld16(g.dl, y);
  tc::tmem_ld_wait();
}

template <int MODE>
struct Need {
  static constexpr bool wo = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool u3 = (MODE == kModeSamplePdf || MODE == kModeQuery);
  static constexpr bool brdf = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool samp = (MODE == kModeSamplePdf || MODE == kModeQuery);
};

// Stage one tile's inputs into `ib`: TMA for full tiles (leader), direct
// per-row copies for the partial last tile.  Returns true if TMA was used.
template <int MODE>
__device__ __forceinline__ bool stage_inputs(const QueryArgs& a, int64_t tile, InBuf& ib,
                                             uint64_t* bar, int r, bool leader) {
  const int64_t q0 = tile * kTile;
  if (q0 + kTile <= a.n) {
    if (leader) {
      uint32_t bytes = kTile * (8 + 4 + 12);
      if (a.lod_stride) bytes += kTile * 4;
      if (Need<MODE>::wo) bytes += kTile * 12;
      if (Need<MODE>::u3) bytes += kTile * 12;
      tc::mbar_arrive_expect_tx(bar, bytes);
      tc::tma_load_1d(tc::smem_u32(ib.uv), a.uv + 2 * q0, kTile * 8, bar);
      if (a.lod_stride) tc::tma_load_1d(tc::smem_u32(ib.lod), a.lod + q0, kTile * 4, bar);
      tc::tma_load_1d(tc::smem_u32(ib.urr), a.u_rr + q0, kTile * 4, bar);
      tc::tma_load_1d(tc::smem_u32(ib.wi), a.wi + 3 * q0, kTile * 12, bar);
      if (Need<MODE>::wo) tc::tma_load_1d(tc::smem_u32(ib.wo), a.wo + 3 * q0, kTile * 12, bar);
      if (Need<MODE>::u3) tc::tma_load_1d(tc::smem_u32(ib.u3), a.u3 + 3 * q0, kTile * 12, bar);
    }
    return true;
  }
  const int64_t q = q0 + r;
  const bool v = q < a.n;
  ib.uv[2 * r] = v ? a.uv[2 * q] : 0.f;
  ib.uv[2 * r + 1] = v ? a.uv[2 * q + 1] : 0.f;
  if (a.lod_stride) ib.lod[r] = v ? a.lod[q] : 0.f;
  ib.urr[r] = v ? a.u_rr[q] : 0.f;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    ib.wi[3 * r + k] = v ? a.wi[3 * q + k] : (k == 2 ? 1.f : 0.f);
    if (Need<MODE>::wo) ib.wo[3 * r + k] = v ? a.wo[3 * q + k] : (k == 2 ? 1.f : 0.f);
    if (Need<MODE>::u3) ib.u3[3 * r + k] = v ? a.u3[3 * q + k] : 0.f;
  }
  return false;
}

// (c): level + taps of one row, texel gathers into SMEM
__device__ __forceinline__ void prefetch_texels(const MatParams& mp, const QueryArgs& a,
                                                const InBuf& ib, GroupSmem& gs, int r,
                                                float lod0) {
  const float u = ib.uv[2 * r], v = ib.uv[2 * r + 1];
  const float lod = a.lod_stride ? ib.lod[r] : lod0;
  const int level = choose_level(mp, lod, ib.urr[r]);
  const Taps t = make_taps(mp, level, u, v);
  gs.aux[r] = make_float4(t.fx, t.fy, __int_as_float(level), 0.f);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    tc::cp_async16(tc::smem_u32(&gs.tex[k * kTile + r]), mp.latent + tap_index(t, k));
}

template <int MODE, int NF, int BW, int BNH, int SW, int SNH, int G>
__global__ void __launch_bounds__(G * 128, 1)
fast_kernel(const __grid_constant__ MatParams mp, const __grid_constant__ QueryArgs a,
            const __grid_constant__ FastConsts fc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mma_bar[G];
  __shared__ uint64_t in_bar[G][2];
  __shared__ uint32_t tbase_sh;
  const int tid = threadIdx.x;
  const int gi = tid / 128, r = tid % 128;
  const int warp = tid / 32;
  constexpr int DW = (BW > SW ? BW : SW) < 16 ? 16 : (BW > SW ? BW : SW);
  constexpr uint32_t kGroupCols = 2 * DW;
  constexpr uint32_t kBiasCol = G * kGroupCols;
  static_assert(kBiasCol + 32 <= 512, "TMEM budget");

  const uint32_t wbytes = (mp.wblob_bytes + 127) & ~127u;
  GroupSmem* gsm = reinterpret_cast<GroupSmem*>(smem + wbytes);
  GroupSmem& gs = gsm[gi];

  // --- CTA setup --------------------------------------------------------------
  {
    const uint4* src = mp.wblob;
    uint4* dst = reinterpret_cast<uint4*>(smem);
    for (uint32_t i = tid; i < mp.wblob_bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  if (tid < G) {
    tc::mbar_init(&mma_bar[tid], 1);
    tc::mbar_init(&in_bar[tid][0], 1);
    tc::mbar_init(&in_bar[tid][1], 1);
  }
  if (warp == 0) tc::tmem_alloc<512>(&tbase_sh);
  tc::fence_proxy_async_smem();
  tc::fence_mbar_init();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = tbase_sh;
  if (warp < 4) {  // bias chunks: (beta_j hi, beta_j lo, 0 ...) for j = 0..3
    const uint32_t lane = (uint32_t)(warp * 32) << 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t v[8] = {fc.beta[j], 0u, 0u, 0u, 0u, 0u, 0u, 0u};
      tc::tmem_st8(tb + lane + kBiasCol + 8 * j, v);
    }
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  FG g;
  g.d0 = tb + gi * kGroupCols;
  g.a0 = g.d0 + DW;
  const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;
  g.dl = g.d0 + lane;
  g.al = g.a0 + lane;
  g.bias0 = tb + kBiasCol;
  g.bar = &mma_bar[gi];
  g.ph = 0;
  g.bar_id = 1 + gi;
  g.wsm = tc::smem_u32(smem);
  g.leader = (r == 0);

  const float lod0 = a.lod_stride ? 0.f : __ldg(a.lod);
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  const int64_t stride = (int64_t)gridDim.x * G;
  int64_t t = (int64_t)blockIdx.x * G + gi;
  uint32_t ph_bits = 0u;   // bit b: mbarrier parity of input buffer b
  uint32_t tma_bits = 0u;  // bit b: buffer b was filled by TMA (wait on its mbarrier)

  // --- prologue: inputs of t and t+s, texels of t ------------------------------
  if (t < ntiles) {
    tma_bits = stage_inputs<MODE>(a, t, gs.in[0], &in_bar[gi][0], r, g.leader) ? 1u : 0u;
    if (t + stride < ntiles)
      tma_bits |= stage_inputs<MODE>(a, t + stride, gs.in[1], &in_bar[gi][1], r, g.leader) ? 2u : 0u;
    if (tma_bits & 1u) {
      tc::mbar_wait(&in_bar[gi][0], 0u);
      ph_bits ^= 1u;
    }
    prefetch_texels(mp, a, gs.in[0], gs, r, lod0);
  }
  tc::cp_async_commit();

  for (int it = 0; t < ntiles; ++it, t += stride) {
    const int b = it & 1;
    InBuf& ib = gs.in[b];
    const int64_t q = t * kTile + r;
    const bool valid = q < a.n;

    // (a) this tile's inputs
    const V3 wi = v3(ib.wi[3 * r], ib.wi[3 * r + 1], ib.wi[3 * r + 2]);
    V3 wo = v3(0.f, 0.f, 1.f), u3 = v3(0.f, 0.f, 0.f);
    if constexpr (Need<MODE>::wo) wo = v3(ib.wo[3 * r], ib.wo[3 * r + 1], ib.wo[3 * r + 2]);
    if constexpr (Need<MODE>::u3) u3 = v3(ib.u3[3 * r], ib.u3[3 * r + 1], ib.u3[3 * r + 2]);

    // (b) blend this tile's texels
    tc::cp_async_wait<0>();
    const float4 aux = gs.aux[r];
    uint4 tex[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) tex[k] = gs.tex[k * kTile + r];
    float z[8];
    blend4(z, tex, aux.x, aux.y);
    if (valid && a.level) a.level[q] = __float_as_int(aux.z);

    // (c) next tile: wait its inputs, gather its texels
    const int64_t t1 = t + stride;
    if (t1 < ntiles) {
      if ((tma_bits >> (b ^ 1)) & 1u) {
        tc::mbar_wait(&in_bar[gi][b ^ 1], (ph_bits >> (b ^ 1)) & 1u);
        ph_bits ^= 1u << (b ^ 1);
      }
      prefetch_texels(mp, a, gs.in[b ^ 1], gs, r, lod0);
    }
    tc::cp_async_commit();

    // after the first barrier of this tile every thread has consumed `ib`:
    // refill it with tile t + 2s
    const int64_t t2 = t + 2 * stride;
    bool direct_next = false;
    auto refill = [&]() {
      if (t2 < ntiles && (t2 + 1) * kTile <= a.n)
        stage_inputs<MODE>(a, t2, ib, &in_bar[gi][b], r, true);
    };
    if (t2 < ntiles && (t2 + 1) * kTile > a.n) direct_next = true;

    bool first_mma = true;
    // (d)+(e) BRDF decode
    if constexpr (Need<MODE>::brdf) {
      {  // frame layer: [fp16(z), 1, 0...]
        uint32_t x[8] = {pack2(z[0], z[1]), pack2(z[2], z[3]), pack2(z[4], z[5]),
                         pack2(z[6], z[7]), 0x00003C00u, 0u, 0u, 0u};
        tc::tmem_st8(g.al, x);
      }
      mma_layer<16, 1, false>(g, mp.layers[mp.frame_layer].b_off, 0, refill);
      first_mma = false;
      uint32_t rr[16];
      tc::tmem_ld16(g.dl, rr);
      tc::tmem_ld_wait();
      float raw[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) raw[k] = __uint_as_float(rr[k]);
      float ti[6], to[6];
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const Frame fr = frame_from_raw(raw + 6 * f);
        ti[3 * f + 0] = dot(fr.t, wi);
        ti[3 * f + 1] = dot(fr.b, wi);
        ti[3 * f + 2] = dot(fr.n, wi);
        to[3 * f + 0] = dot(fr.t, wo);
        to[3 * f + 1] = dot(fr.b, wo);
        to[3 * f + 2] = dot(fr.n, wo);
      }
      static_assert(NF == 2, "fast path: two frames");
      // decoder input [z, T wi, T wo, 1] (K = 32)
      uint32_t x[16] = {pack2(z[0], z[1]), pack2(z[2], z[3]), pack2(z[4], z[5]), pack2(z[6], z[7]),
                        pack2(ti[0], ti[1]), pack2(ti[2], ti[3]), pack2(ti[4], ti[5]),
                        pack2(to[0], to[1]), pack2(to[2], to[3]), pack2(to[4], to[5]),
                        0x00003C00u, 0u, 0u, 0u, 0u, 0u};
      tc::tmem_st16(g.al, x);
      uint32_t y[16];
      run_chain<BW, BNH, 2>(g, mp, mp.brdf_first, NoOp{}, y);
      if (valid) {
        const bool up = (wi.z > 0.f) && (wo.z > 0.f);
        const float s = fc.inv_brdf;
        const V3 f = up ? v3(brdf_output(__uint_as_float(y[0]) * s),
                             brdf_output(__uint_as_float(y[1]) * s),
                             brdf_output(__uint_as_float(y[2]) * s))
                        : v3(0.f, 0.f, 0.f);
        stg3(a.rgb, q, f);
        if (mp.albedo && a.albedo) {
          const V3 al = up ? v3(fmaxf(__uint_as_float(y[3]) * s, 0.f),
                                fmaxf(__uint_as_float(y[4]) * s, 0.f),
                                fmaxf(__uint_as_float(y[5]) * s, 0.f))
                           : v3(0.f, 0.f, 0.f);
          stg3(a.albedo, q, al);
        }
      }
    }
    if constexpr (Need<MODE>::samp) {
      uint32_t x[8] = {pack2(z[0], z[1]), pack2(z[2], z[3]), pack2(z[4], z[5]), pack2(z[6], z[7]),
                       pack2(wi.x, wi.y), pack2(wi.z, 1.f), 0u, 0u};
      tc::tmem_st8(g.al, x);
      uint32_t y[16];
      if (first_mma) run_chain<SW, SNH, 1>(g, mp, mp.samp_first, refill, y);
      else run_chain<SW, SNH, 1>(g, mp, mp.samp_first, NoOp{}, y);
      float raw[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) raw[k] = __uint_as_float(y[k]);
      const Proxy p = proxy_from_raw(raw, mp.isotropic != 0, fc.inv_samp);
      if (valid) {
        if (a.params9) store_proxy(a.params9, q, p);
        const V3 s = proxy_sample(p, wi, u3.x, u3.y, u3.z);
        stg3(a.ws, q, s);
        a.pdf[q] = proxy_pdf(p, wi, s);
      }
    }
    // partial last tile t2: every thread copies its own row (no TMA)
    if (direct_next) stage_inputs<MODE>(a, t2, ib, &in_bar[gi][b], r, false);
    tma_bits = (tma_bits & ~(1u << b)) | (((t2 < ntiles) && !direct_next) ? (1u << b) : 0u);
  }

  tc::cp_async_wait<0>();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_free<512>(tb);
}

uint32_t fp16_bits(double v) {
  const __half h = __double2half(v);
  return *reinterpret_cast<const uint16_t*>(&h);
}

FastConsts make_consts(int brdf_nh, int samp_nh) {
  FastConsts c{};
  const double cc = 1.0 + (double)kLk;
  for (int j = 0; j < 4; ++j) {
    const double beta = std::pow(cc, j);
    const uint32_t hi = fp16_bits(beta);
    const __half hh = *reinterpret_cast<const __half*>(&hi);
    const double rem = beta - (double)__half2float(hh);
    c.beta[j] = hi | (fp16_bits(rem) << 16);
  }
  c.inv_brdf = (float)(1.0 / std::pow(cc, brdf_nh));
  c.inv_samp = (float)(1.0 / std::pow(cc, samp_nh));
  return c;
}

int g_sms = 0;

template <int MODE, int NF, int BW, int BNH, int SW, int SNH, int G>
cudaError_t launch_fast_t(const MatParams& mp, const QueryArgs& a, cudaStream_t s) {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  auto kern = fast_kernel<MODE, NF, BW, BNH, SW, SNH, G>;
  const int smem = (int)(((mp.wblob_bytes + 127) & ~127u) + G * sizeof(GroupSmem));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  int64_t grid = g_sms;
  if (grid > (ntiles + G - 1) / G) grid = (ntiles + G - 1) / G;
  if (grid < 1) grid = 1;
  const FastConsts fc = make_consts(BNH, SNH);
  kern<<<(int)grid, G * 128, smem, s>>>(mp, a, fc);
  ++g_launches;
  return cudaGetLastError();
}

template <int NF, int BW, int BNH, int SW, int SNH, int G>
cudaError_t launch_fast_arch(int mode, const MatParams& mp, const QueryArgs& a, cudaStream_t s) {
  switch (mode) {
    case kModeEval: return launch_fast_t<kModeEval, NF, BW, BNH, SW, SNH, G>(mp, a, s);
    case kModeSamplePdf: return launch_fast_t<kModeSamplePdf, NF, BW, BNH, SW, SNH, G>(mp, a, s);
    case kModeQuery: return launch_fast_t<kModeQuery, NF, BW, BNH, SW, SNH, G>(mp, a, s);
    default: return cudaErrorNotSupported;
  }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

// Returns cudaErrorNotSupported when the fast path does not apply (caller
// then uses the generic kernel).
cudaError_t launch_fast(const MatParams& mp, int mode, const QueryArgs& a, cudaStream_t s) {
  if (mp.fast_arch < 0 || mp.texel_fp32 || a.idx) return cudaErrorNotSupported;
  if (mode != kModeEval && mode != kModeSamplePdf && mode != kModeQuery)
    return cudaErrorNotSupported;
  if (!aligned16(a.uv) || !aligned16(a.u_rr) || !aligned16(a.wi) ||
      (a.lod_stride && !aligned16(a.lod)) || (a.wo && !aligned16(a.wo)) ||
      (a.u3 && !aligned16(a.u3)))
    return cudaErrorNotSupported;
  switch (mp.fast_arch) {
    case 0: return launch_fast_arch<2, 32, 2, 32, 3, 6>(mode, mp, a, s);
    case 1: return launch_fast_arch<2, 16, 2, 32, 3, 6>(mode, mp, a, s);
    case 2: return launch_fast_arch<2, 64, 3, 32, 3, 3>(mode, mp, a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace nmq
