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
#include <cstdlib>
#include "tc.cuh"
#include "nmq_device.cuh"
#include "nmq_internal.h"

namespace nmq {
namespace {

using namespace dev;

#ifndef NMQ_FAST_G
#define NMQ_FAST_G 5  // tile groups per CTA for hidden width <= 32 (SMEM: 5 max)
#endif

constexpr float kLk = 0.98019802570343017578f;  // fp32(99/101)

struct FastConsts {
  uint32_t beta[4];  // fp16 (hi | lo << 16) of c^j
  float inv_brdf;    // 1 / c^(brdf leaky layers)
  float inv_samp;    // 1 / c^(sampler leaky layers)
};

template <int MODE>
struct Need {
  static constexpr bool wo = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool u3 = (MODE == kModeSamplePdf || MODE == kModeQuery);
  static constexpr bool brdf = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool samp = (MODE == kModeSamplePdf || MODE == kModeQuery);
};

// per-group SMEM staging of one tile's inputs (kept small: the rest of the
// SM's 228 KB stays L1, which serves the coarse pyramid levels)
template <int MODE>
struct alignas(16) InBuf {
  float uv[2 * kTile];
  float lod[kTile];
  float urr[kTile];
  float wi[3 * kTile];
  float wo[Need<MODE>::wo ? 3 * kTile : 4];
  float u3[Need<MODE>::u3 ? 3 * kTile : 4];
};
template <int MODE>
struct GroupSmem {
  InBuf<MODE> in[2];  // double-buffered inputs (TMA, 2 tiles ahead)
};

// Optional per-phase cycle accounting (-DNMQ_TRACE): work / barrier /
// issue / overlap / mma-wait buckets per warp of each tile group.
#ifdef NMQ_TRACE
__device__ unsigned long long g_trace[64];
#define TR(g, k)                          \
  do {                                    \
    const long long now_ = clock64();     \
    (g).tr[k] += now_ - (g).tr_prev;      \
    (g).tr_prev = now_;                   \
  } while (0)
#else
#define TR(g, k) \
  do {           \
  } while (0)
#endif
enum { kTrWork = 0, kTrBar = 1, kTrIssue = 2, kTrOverlap = 3, kTrWait = 4, kTrN = 5 };

struct FG {
#ifdef NMQ_TRACE
  long long tr[kTrN];
  long long tr_prev;
#endif
  uint32_t dl, al;    // TMEM addresses with this warp's lane field (ld/st)
  uint32_t d0, a0;    // lane-0 TMEM addresses (MMA operands)
  uint32_t bias0;     // bias chunk j at bias0 + 8j
  uint64_t desc0;     // SMEM descriptor of the weight blob base (SBO = 128)
  uint64_t* bar;
  uint32_t ph;
  uint32_t bar_id;    // named barrier: all 128 threads before an MMA issue
  uint32_t done_id;   // named barrier: MMA completion, signalled by warp 0
  bool leader;        // thread 0 of the group: issues the MMAs
  bool warp0;         // warp 0 of the group: polls the MMA mbarrier
};

__device__ __forceinline__ void split_scaled(uint32_t ra, uint32_t rb, uint32_t& hi, uint32_t& lo) {
  // a~ = y + k|y| for the pair (one FFMA2 with the |.| modifier), then
  // (hi, lo) fp16 with hi + lo = a~ to ~2^-22
  const float2 ab = __ffma2_rn(make_float2(fabsf(__uint_as_float(ra)), fabsf(__uint_as_float(rb))),
                               make_float2(kLk, kLk),
                               make_float2(__uint_as_float(ra), __uint_as_float(rb)));
  const float a = ab.x, b = ab.y;
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

// Issue one MMA layer (all 128 threads of the group call; the leader issues
// KA k-steps against A in TMEM, + the bias chunk when HID).  `hook` runs on
// the leader right after issue (used to launch input TMA once every thread
// has passed the barrier).  The caller overlaps independent work before
// mma_wait().
template <int N, int KA, bool HID, class F>
__device__ __forceinline__ void mma_issue(FG& g, uint32_t b_off, int bias_chunk, F&& hook) {
  TR(g, kTrWork);
  tc::tmem_st_wait();
  tc::tc_fence_before();
  tc::named_bar(g.bar_id, 128);
  TR(g, kTrBar);
  if (g.leader) {
    tc::tc_fence_after();
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    constexpr uint32_t lbo = N * 16;
    // descriptor = base + (LBO field) + start offset (all fields linear, no carries)
    const uint64_t d = g.desc0 + ((uint64_t)(lbo >> 4) << 16) + (b_off >> 4);
#pragma unroll
    for (int s = 0; s < KA; ++s) tc::mma_ts(g.d0, g.a0 + 8 * s, d + ((s * 2 * lbo) >> 4), idesc, s > 0);
    if constexpr (HID)
      tc::mma_ts(g.d0, g.bias0 + 8 * bias_chunk, d + ((KA * 2 * lbo) >> 4), idesc, 1);
    tc::mma_commit(g.bar);
  }
  hook();  // every thread; the hook selects its own issuing thread
  TR(g, kTrIssue);
}
// MMA completion: warp 0 polls the mbarrier, then releases the other three
// warps, which sleep on a named barrier (one instruction each).
__device__ __forceinline__ void mma_wait(FG& g) {
  TR(g, kTrOverlap);
  if (g.warp0) {
    tc::mbar_wait(g.bar, g.ph);
    asm volatile("bar.arrive %0, %1;" ::"r"(g.done_id), "r"(128) : "memory");
  } else {
    tc::named_bar(g.done_id, 128);
  }
  g.ph ^= 1u;
  tc::tc_fence_after();
  TR(g, kTrWait);
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

// chain: first layer (input already in A) + (NH-1) hidden + output (N=16).
//   lead          leader-only, right after the first layer is issued
//   first_overlap all threads, while the first layer's MMA runs
//   last_overlap  all threads, while the output layer's MMA runs
template <int W, int NH, int KA0, class L, class F1, class F2>
__device__ __forceinline__ void run_chain(FG& g, const MatParams& mp, int first, L&& lead,
                                          F1&& first_overlap, F2&& last_overlap,
                                          uint32_t (&y)[16]) {
  mma_issue<W, KA0, false>(g, mp.layers[first].b_off, 0, lead);
  first_overlap();
  mma_wait(g);
#pragma unroll
  for (int i = 1; i < NH; ++i) {
    hidden_epi<W>(g);
    mma_issue<W, 2 * W / 16, true>(g, mp.layers[first + i].b_off, i, NoOp{});
    mma_wait(g);
  }
  hidden_epi<W>(g);
  mma_issue<16, 2 * W / 16, true>(g, mp.layers[first + NH].b_off, NH, NoOp{});
  last_overlap();
  mma_wait(g);
  tc::tmem_ld16(g.dl, y);
  tc::tmem_ld_wait();
}

// Stage one tile's inputs into `ib`: TMA bulk copies for full tiles (issued
// by one thread), direct per-row copies for the partial last tile.
// Returns true if TMA was used (consumers then wait on `bar`).
template <int MODE>
__device__ __forceinline__ bool stage_inputs(const QueryArgs& a, int tile, InBuf<MODE>& ib,
                                             uint64_t* bar, int r, bool issuer) {
  const int64_t q0 = (int64_t)tile * kTile;
  if (q0 + kTile <= a.n) {
    if (issuer) {
      uint32_t bytes = kTile * (8 + 4 + 12);
      if (a.lod_stride) bytes += kTile * 4;
      if (Need<MODE>::wo) bytes += kTile * 12;
      if (Need<MODE>::u3) bytes += kTile * 12;
      tc::mbar_arrive_expect_tx(bar, bytes);
      tc::tma_load_1d(tc::smem_u32(ib.uv), a.uv + 2 * q0, kTile * 8, bar);
      if (a.lod_stride) tc::tma_load_1d(tc::smem_u32(ib.lod), a.lod + q0, kTile * 4, bar);
      tc::tma_load_1d(tc::smem_u32(ib.urr), a.u_rr + q0, kTile * 4, bar);
      tc::tma_load_1d(tc::smem_u32(ib.wi), a.wi + 3 * q0, kTile * 12, bar);
      if constexpr (Need<MODE>::wo)
        tc::tma_load_1d(tc::smem_u32(ib.wo), a.wo + 3 * q0, kTile * 12, bar);
      if constexpr (Need<MODE>::u3)
        tc::tma_load_1d(tc::smem_u32(ib.u3), a.u3 + 3 * q0, kTile * 12, bar);
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
    if constexpr (Need<MODE>::wo) ib.wo[3 * r + k] = v ? a.wo[3 * q + k] : (k == 2 ? 1.f : 0.f);
    if constexpr (Need<MODE>::u3) ib.u3[3 * r + k] = v ? a.u3[3 * q + k] : 0.f;
  }
  return false;
}

// Texel prefetch into registers: level + taps of one row and the 4 texel
// loads (LDG.128, L1-cached: the coarse pyramid levels live in L1).  Issued
// a full tile ahead of use, so the loads land while the current tile runs.
struct TexPrefetch {
  uint4 tex[4];
  float fx, fy;
  int level;
};

template <int MODE>
__device__ __forceinline__ void prefetch_texels(const MatParams& mp, const QueryArgs& a,
                                                const InBuf<MODE>& ib, int r, float lod0,
                                                TexPrefetch& p) {
  const float u = ib.uv[2 * r], v = ib.uv[2 * r + 1];
  const float lod = a.lod_stride ? ib.lod[r] : lod0;
  p.level = choose_level(mp, lod, ib.urr[r]);
  const Taps t = make_taps(mp, p.level, u, v);
  p.fx = t.fx;
  p.fy = t.fy;
#pragma unroll
  for (int k = 0; k < 4; ++k) p.tex[k] = __ldg(mp.latent + tap_index(t, k));
}

// Per-row state of one tile (blended latent code + level).
struct TileZ {
  float2 z[4];  // channel pairs
  int level;
};

__device__ __forceinline__ void blend_prefetched(const TexPrefetch& p, TileZ& o) {
  blend4x2(o.z, p.tex, p.fx, p.fy);
  o.level = p.level;
}

// frame layer 8 -> 12 on the CUDA cores: raw = W fp16(z) + b with packed
// FFMA2 and weights from the constant bank (exact fp32 like the reference).
__device__ __forceinline__ void frame_layer_simt(const MatParams& mp, const uint32_t (&zp)[4],
                                                 float (&raw)[12]) {
  float zh[8];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&zp[c]));
    zh[2 * c] = f.x;
    zh[2 * c + 1] = f.y;
  }
#pragma unroll
  for (int p = 0; p < 6; ++p) {
    float2 acc = mp.fb[p];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = fma2s(mp.fw[p][k], zh[k], acc);
    raw[2 * p] = acc.x;
    raw[2 * p + 1] = acc.y;
  }
}

// BRDF output layer W -> 3 (6 with albedo) on the CUDA cores from the last
// hidden layer's scaled pre-activations in D: a~ = P + k|P| (FFMA2), then
// y_j = (sum_k w_jk a~_k) / c^depth + b_j.
template <int W>
__device__ __forceinline__ void out_layer_simt(const FG& g, const MatParams& mp, float inv_scale,
                                               bool albedo, float (&y)[6]) {
  float2 av[W / 2];
#pragma unroll
  for (int c0 = 0; c0 < W; c0 += 32) {
    constexpr int kChunk = W < 32 ? W : 32;
    uint32_t r[32];
    if constexpr (W == 16) {
      uint32_t r16[16];
      tc::tmem_ld16(g.dl, r16);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = r16[i];
    } else {
      tc::tmem_ld32(g.dl + c0, r);
      tc::tmem_ld_wait();
    }
#pragma unroll
    for (int i = 0; i < kChunk / 2; ++i) {
      const float2 p = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
      av[c0 / 2 + i] = __ffma2_rn(make_float2(fabsf(p.x), fabsf(p.y)), make_float2(kLk, kLk), p);
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    float2 acc = mul2(mp.ow[j][0], av[0]);
#pragma unroll
    for (int q = 1; q < W / 2; ++q) acc = fma2(mp.ow[j][q], av[q], acc);
    y[j] = fmaf(acc.x + acc.y, inv_scale, mp.ob[j]);
  }
  if (albedo) {  // warp-uniform branch: the albedo head costs nothing otherwise
#pragma unroll
    for (int j = 3; j < 6; ++j) {
      float2 acc = mul2(mp.ow[j][0], av[0]);
#pragma unroll
      for (int q = 1; q < W / 2; ++q) acc = fma2(mp.ow[j][q], av[q], acc);
      y[j] = fmaf(acc.x + acc.y, inv_scale, mp.ob[j]);
    }
  } else {
    y[3] = y[4] = y[5] = 0.f;
  }
}

// BRDF chain of the specialized kernel: first layer (input in A, KA0 k-steps)
// + (NH-1) hidden layers on the tensor cores; output layer on the CUDA cores.
template <int W, int NH, int KA0, class L, class F1, class F2>
__device__ __forceinline__ void brdf_chain(FG& g, const MatParams& mp, float inv_scale,
                                           L&& lead, F1&& first_overlap, F2&& last_overlap,
                                           float (&y)[6]) {
  mma_issue<W, KA0, false>(g, mp.layers[mp.brdf_first].b_off, 0, lead);
  if constexpr (NH == 1) {
    first_overlap();
    last_overlap();
  } else {
    first_overlap();
  }
  mma_wait(g);
#pragma unroll
  for (int i = 1; i < NH; ++i) {
    hidden_epi<W>(g);
    mma_issue<W, 2 * W / 16, true>(g, mp.layers[mp.brdf_first + i].b_off, i, NoOp{});
    if (i == NH - 1) last_overlap();
    mma_wait(g);
  }
  out_layer_simt<W>(g, mp, inv_scale, mp.albedo != 0, y);
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
  // warp-uniform by construction (shfl from lane 0): lets ptxas keep the
  // TMEM/MMA operands in uniform registers (no R2UR waterfall per MMA)
  const int gi = __shfl_sync(0xffffffffu, tid / 128, 0), r = tid % 128;
  const int warp = tid / 32;
  constexpr int DW = (BW > SW ? BW : SW) < 16 ? 16 : (BW > SW ? BW : SW);
  constexpr uint32_t kGroupCols = 2 * DW;
  constexpr uint32_t kBiasCol = G * kGroupCols;
  static_assert(kBiasCol + 32 <= 512, "TMEM budget");
  static_assert(NF == 2, "fast path: two learned frames");
  // power-of-two allocation covering all groups + bias chunks, so CTAs that
  // happen to share an SM never block each other in tcgen05.alloc
  constexpr uint32_t kTmemCols = kBiasCol + 32 <= 128 ? 128 : (kBiasCol + 32 <= 256 ? 256 : 512);

  const uint32_t wbytes = (mp.wblob_bytes + 127) & ~127u;
  GroupSmem<MODE>* gsm = reinterpret_cast<GroupSmem<MODE>*>(smem + wbytes);
  GroupSmem<MODE>& gs = gsm[gi];

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
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tbase_sh);
  tc::fence_proxy_async_smem();
  tc::fence_mbar_init();
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tbase_sh, 0);
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
  g.done_id = 1 + G + gi;
  static_assert(1 + 2 * G <= 16, "named barriers");
  g.desc0 = tc::smem_desc(tc::smem_u32(smem), 0, 128);
  g.leader = (r == 0);
  g.warp0 = (r < 32);
  const bool tma_thread = (r == 32);  // input TMA off the MMA-issuing thread
#ifdef NMQ_TRACE
  for (int k = 0; k < kTrN; ++k) g.tr[k] = 0;
  g.tr_prev = clock64();
#endif

  const float lod0 = a.lod_stride ? 0.f : __ldg(a.lod);
  const int ntiles = (int)((a.n + kTile - 1) / kTile);  // host guarantees < 2^31
  const int last_full = (int)(a.n / kTile);                // tiles [0, last_full) are full
  const int stride = gridDim.x * G;
  int t = blockIdx.x * G + gi;
  uint32_t ph_bits = 0u;   // bit b: mbarrier parity of input buffer b
  uint32_t tma_bits = 0u;  // bit b: input buffer b was filled by TMA

  auto wait_in = [&](int b) {
    if ((tma_bits >> b) & 1u) {
      tc::mbar_wait(&in_bar[gi][b], (ph_bits >> b) & 1u);
      ph_bits ^= 1u << b;
    }
  };

  // --- prologue: stage t and t+s, fetch + blend t --------------------------------
  TileZ cur;
  if (t < ntiles) {
    tma_bits = stage_inputs<MODE>(a, t, gs.in[0], &in_bar[gi][0], r, tma_thread) ? 1u : 0u;
    if (t + stride < ntiles)
      tma_bits |=
          stage_inputs<MODE>(a, t + stride, gs.in[1], &in_bar[gi][1], r, tma_thread) ? 2u : 0u;
    wait_in(0);
    TexPrefetch p0;
    prefetch_texels<MODE>(mp, a, gs.in[0], r, lod0, p0);
    blend_prefetched(p0, cur);
  }

  for (int it = 0; t < ntiles; ++it, t += stride) {
    const int b = it & 1;
    const InBuf<MODE>& ib = gs.in[b];
    const int64_t q = (int64_t)t * kTile + r;
    const bool valid = q < a.n;
    const int t1 = t + stride, t2 = t + 2 * stride;
    const bool direct2 = t2 < ntiles && t2 >= last_full;
    if (valid && a.level) a.level[q] = cur.level;

    // next tile's texels: issued now, blended at the end of this iteration
    TexPrefetch nx;
    if (t1 < ntiles) {
      wait_in(b ^ 1);
      prefetch_texels<MODE>(mp, a, gs.in[b ^ 1], r, lod0, nx);
    }
    // this tile's directions (buffer b is refilled after the first barrier)
    const V3 wi = v3(ib.wi[3 * r], ib.wi[3 * r + 1], ib.wi[3 * r + 2]);
    V3 wo = v3(0.f, 0.f, 1.f), u3 = v3(0.f, 0.f, 0.f);
    if constexpr (Need<MODE>::wo) wo = v3(ib.wo[3 * r], ib.wo[3 * r + 1], ib.wo[3 * r + 2]);
    if constexpr (Need<MODE>::u3) u3 = v3(ib.u3[3 * r], ib.u3[3 * r + 1], ib.u3[3 * r + 2]);

    auto lead = [&]() {  // after the first barrier: refill buffer b with tile t2
      if (tma_thread && t2 < ntiles && !direct2)
        stage_inputs<MODE>(a, t2, gs.in[b], &in_bar[gi][b], r, true);
    };

    uint32_t zp[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) zp[c] = pack2(cur.z[c].x, cur.z[c].y);

    bool leaded = false;
    if constexpr (Need<MODE>::brdf) {
      float raw[12];
      frame_layer_simt(mp, zp, raw);
      float ti[6], to[6];
      frames2_transform(raw, wi, wo, ti, to);
      // decoder input [z, T wi, T wo, 1] (K = 32)
      const uint32_t x[16] = {zp[0], zp[1], zp[2], zp[3],
                              pack2(ti[0], ti[1]), pack2(ti[2], ti[3]), pack2(ti[4], ti[5]),
                              pack2(to[0], to[1]), pack2(to[2], to[3]), pack2(to[4], to[5]),
                              0x00003C00u, 0u, 0u, 0u, 0u, 0u};
      tc::tmem_st16(g.al, x);
      float y[6];
      brdf_chain<BW, BNH, 2>(g, mp, fc.inv_brdf, lead, NoOp{}, NoOp{}, y);
      leaded = true;
      if (valid) {
        const bool up = (wi.z > 0.f) && (wo.z > 0.f);
        const V3 f = up ? v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2]))
                        : v3(0.f, 0.f, 0.f);
        stg3(a.rgb, q, f);
        if (mp.albedo && a.albedo) {
          const V3 al = up ? v3(fmaxf(y[3], 0.f), fmaxf(y[4], 0.f), fmaxf(y[5], 0.f))
                           : v3(0.f, 0.f, 0.f);
          stg3(a.albedo, q, al);
        }
      }
    }
    if constexpr (Need<MODE>::samp) {
      const uint32_t x[8] = {zp[0], zp[1], zp[2], zp[3],
                             pack2(wi.x, wi.y), pack2(wi.z, 1.f), 0u, 0u};
      tc::tmem_st8(g.al, x);
      uint32_t y[16];
      if (leaded) run_chain<SW, SNH, 1>(g, mp, mp.samp_first, NoOp{}, NoOp{}, NoOp{}, y);
      else run_chain<SW, SNH, 1>(g, mp, mp.samp_first, lead, NoOp{}, NoOp{}, y);
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
    if (direct2) stage_inputs<MODE>(a, t2, gs.in[b], &in_bar[gi][b], r, false);
    tma_bits = (tma_bits & ~(1u << b)) | ((t2 < ntiles && !direct2) ? (1u << b) : 0u);
    if (t1 < ntiles) blend_prefetched(nx, cur);
  }

  TR(g, kTrWork);
#ifdef NMQ_TRACE
  if ((r & 31) == 0)
    for (int k = 0; k < kTrN; ++k) atomicAdd(&g_trace[(r >> 5) * 8 + k], (unsigned long long)g.tr[k]);
#endif
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_free<kTmemCols>(tb);
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
  const int smem = (int)(((mp.wblob_bytes + 127) & ~127u) + G * sizeof(GroupSmem<MODE>));
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

#ifdef NMQ_TRACE
extern "C" int nm_trace_read(unsigned long long* out, int n, int reset) {
  if (n > 64) n = 64;
  cudaMemcpyFromSymbol(out, g_trace, n * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[64] = {0};
    cudaMemcpyToSymbol(g_trace, z, sizeof(z));
  }
  return 0;
}
#endif

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
    case 0:
#ifdef NMQ_G_SWEEP  // experiment build: tile groups per CTA from $NMQ_G
      switch (getenv("NMQ_G") ? atoi(getenv("NMQ_G")) : NMQ_FAST_G) {
        case 1: return launch_fast_arch<2, 32, 2, 32, 3, 1>(mode, mp, a, s);
        case 2: return launch_fast_arch<2, 32, 2, 32, 3, 2>(mode, mp, a, s);
        case 3: return launch_fast_arch<2, 32, 2, 32, 3, 3>(mode, mp, a, s);
        case 4: return launch_fast_arch<2, 32, 2, 32, 3, 4>(mode, mp, a, s);
        case 5: return launch_fast_arch<2, 32, 2, 32, 3, 5>(mode, mp, a, s);
        case 6: return launch_fast_arch<2, 32, 2, 32, 3, 6>(mode, mp, a, s);
        case 7: return launch_fast_arch<2, 32, 2, 32, 3, 7>(mode, mp, a, s);
        default: break;
      }
#endif
      return launch_fast_arch<2, 32, 2, 32, 3, NMQ_FAST_G>(mode, mp, a, s);
    case 1: return launch_fast_arch<2, 16, 2, 32, 3, NMQ_FAST_G>(mode, mp, a, s);
    case 2: return launch_fast_arch<2, 64, 3, 32, 3, 3>(mode, mp, a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace nmq
