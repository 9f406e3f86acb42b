// nmq_fast.cu — pipelined, architecture-specialized fused query kernels
// (the coherent per-material path).
//
// One persistent CTA per SM holds G tile groups of 128 threads (thread r of
// a group owns row r of its tiles = TMEM lane r).  Each group keeps NS tiles
// in flight ("slots") and walks them through the same stage sequence in
// lock-step, slot by slot:
//
//     for each stage k:  for each slot s:  wait MMA(s, k-1) -> SIMT -> issue MMA(s, k)
//
// so while slot s's MMA runs on the tensor core the group's warps do the
// SIMT stage of slot s+1.  A tile's stages (eval, 2x32):
//
//     0  frame layer D -> frames, T.wi, T.wo (input chunk 1) -> BRDF layer 1;
//        rows whose T.w may round differently from the reference are queued
//     1  scaled leaky + hi/lo split                           -> BRDF layer 2
//     2  BRDF output layer (CUDA cores), rgb store; blend the slot's next
//        tile's prefetched texels -> input chunk 0 -> its frame layer
//
// sample+pdf: 0..2 hidden epilogues -> sampler layers 2..4, 3 proxy /
// sample / pdf + next tile's sampler layer 1; query = eval stages, then the
// sampler's.  The first MMA of a tile is issued by the previous tile's last
// stage, so the chain never starts cold.
//
// Inputs (uv, lod, u_rr, wi, wo, u3) reach SMEM by 1-D TMA bulk copies two
// tiles ahead per slot; each thread's four 16-byte texel loads for the slot's
// next tile are issued at stage 0 (L1-cached LDG.128) and blended — in
// float64, exactly as latent.py:96 — at the last stage.
//
// Hidden activations use the scaled-leaky trick a~ = y + k|y| (k = 99/101)
// = c * leaky(y), c = 1 + k: the scale propagates through the (positively
// homogeneous) network and is undone on the raw outputs; layer biases are
// multiplied by c^depth inside the MMA via an fp16 (hi, lo) pair in the TMEM
// bias chunk.  The exact hi/lo split is F2FP + FHFMA (a - f32(hi)) + F2FP.
//
// Exact rounding of the decoder's direction inputs.  The
// reference computes T.wi / T.wo in float64 from the frame layer's fp32
// outputs, narrows to fp32 and rounds to fp16 (neural.py:282-287).  The
// tensor-core frame layer and the fp32 frames here are within a small,
// conditioning-scaled bound of those values; a row whose fast value lies
// within that bound of an fp16 rounding midpoint is queued (input row, fp16
// latent code, fast fp16 inputs) in a per-CTA region of a global queue.
// After its last tile each CTA resolves its own entries (resolve_entries, in
// the kernel's epilogue; NMQ_RESOLVE_FUSED=0 runs resolve_kernel as a
// follow-up launch instead, measured slower): it recomputes each queued
// row's inputs in the reference's own arithmetic (frame_raw_seq +
// frame_tw64); where an fp16 value differs, the warp re-evaluates the BRDF
// decoder for that row on the CUDA cores (fp32) and overwrites its output.
// Nothing of it sits in the pipelined loop: a call there constrains its
// register allocation (the prefetched texels spill) and an SMEM ring takes
// the L1 the coarse pyramid levels live in (both measured: -40 % / -8 % on
// C2).  NMQ_TW_INLINE=1 computes every row's inputs in float64 inline
// instead (no queue): measured equal on C2 (22.3 G q/s either way).
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include "tc.cuh"
#include "nmq_device.cuh"
#include "nmq_internal.h"

namespace nmq {
namespace {

using namespace dev;

// Tile groups per CTA for hidden width <= 32, per mode (measured on B200:
// more groups hide more latency until registers spill; 7 is the TMEM limit).
#ifndef NMQ_G_EVAL
#define NMQ_G_EVAL 7
#endif
#ifndef NMQ_G_SAMPLE
#define NMQ_G_SAMPLE 7  // with SMEM texel staging (NMQ_TEX_SMEM); 5 with register prefetch
#endif
#ifndef NMQ_G_QUERY
#define NMQ_G_QUERY 5
#endif
#ifndef NMQ_PDL
#define NMQ_PDL 1  // programmatic dependent launch (prologue overlaps the previous kernel's tail): C2 +4 %
#endif
#ifndef NMQ_TW_INLINE
#define NMQ_TW_INLINE 0  // 1: every row's direction inputs in float64 inline (no queue)
#endif
#ifndef NMQ_FAST_NS
#define NMQ_FAST_NS 1  // tiles in flight per group (2 = ping-pong; slower: fewer warps)
#endif

constexpr float kLk = 0.98019802570343017578f;  // fp32(99/101)

// Exact-rounding queue of one launch: CTA b owns the region
// ent[kQueueWords * b * cap, kQueueWords * (b+1) * cap), laid out by word
// (structure of arrays: word w of entry k at region[w * cap + k], so a
// warp's appends and the resolve's loads are coalesced): {row, x16[0..2]},
// {x16[3..5], z16[0]}, {z16[1..3], wi.x}, {wi.y, wi.z, wo.x, wo.y},
// {wo.z, frames to resolve, 0, 0}, {fast rgb (spp-mean launches only), 0};
// it writes how many entries it used to cnt[b] when it exits.
constexpr int kQueueWords = 6;
struct ResolveQ {
  uint4* ent;
  uint32_t* cnt;
  uint32_t cap;
};

struct FastConsts {
  uint32_t beta[4];  // fp16 (hi | lo << 16) of c^j
  float inv_brdf;    // 1 / c^(brdf leaky layers)
  float inv_samp;    // 1 / c^(sampler leaky layers)
  float tw_delta;    // error bound of the fast T.w per unit conditioning
  ResolveQ q;        // BRDF modes
};

template <int MODE>
struct Need {
  static constexpr bool wo = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool u3 = (MODE == kModeSamplePdf || MODE == kModeQuery);
  static constexpr bool brdf = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool samp = (MODE == kModeSamplePdf || MODE == kModeQuery);
};

// per-slot SMEM staging of one tile's inputs
template <int MODE>
struct alignas(16) InBuf {
  float uv[2 * kTile];
  float lod[kTile];
  float urr[kTile];
  float wi[3 * kTile];
  float wo[Need<MODE>::wo ? 3 * kTile : 4];
  float u3[Need<MODE>::u3 ? 3 * kTile : 4];
};

template <int... I, class F>
__device__ __forceinline__ void sfor_impl(std::integer_sequence<int, I...>, F&& f) {
  (f(std::integral_constant<int, I>{}), ...);
}
// compile-time loop: f(integral_constant<int, 0>), ..., f(<N-1>)
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(std::make_integer_sequence<int, N>{}, f);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

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

// Does an fp16 rounding midpoint lie within +-d of either value of the pair?
// (their fp16 roundings of v + d and v - d differ)
__device__ __forceinline__ uint32_t near_mid2(float a, float b, float2 d) {
  const float2 v = make_float2(a, b);
  const float2 up = __ffma2_rn(d, make_float2(1.f, 1.f), v);
  const float2 dn = __ffma2_rn(d, make_float2(-1.f, -1.f), v);
  return pack2(up.x, up.y) ^ pack2(dn.x, dn.y);
}

// Group-wide constants.
struct GG {
  uint32_t bias0;   // TMEM bias chunk j at bias0 + 8j (lane 0)
  uint64_t desc0;   // SMEM descriptor of the weight blob base (SBO = 128)
  uint32_t bar_id;  // named barrier of the group (before every MMA issue)
  int r;            // row of this thread in the group's tiles
};

// MMA completion: every warp sleeps on the mbarrier (try_wait with a suspend hint).
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t& ph) {
  tc::mbar_wait(bar, ph);
  ph ^= 1u;
  tc::tc_fence_after();
}

// One MMA layer: the group's 128 threads finish their TMEM stores and meet
// at the group barrier; lane 0 of warp LW issues KA k-steps of A (TMEM) x B
// (SMEM weights at b_off), + the bias chunk when HID, and commits to `bar`.
// `hook` then runs on every thread (TMA refills after the barrier).
template <int N, int KA, bool HID, int LW, class F>
__device__ __forceinline__ void mma_issue(const GG& g, uint32_t d_tmem, uint32_t a_tmem,
                                          uint32_t b_off, int bias_chunk, uint64_t* bar, F&& hook) {
  tc::tmem_st_wait();
  tc::tc_fence_before();
  tc::named_bar(g.bar_id, 128);
  if (g.r == 32 * LW) {
    tc::tc_fence_after();
    constexpr uint32_t idesc = tc::idesc_f16(128, N);
    constexpr uint32_t lbo = N * 16;
    // descriptor = base + (LBO field) + start offset (all fields linear, no carries)
    const uint64_t d = g.desc0 + ((uint64_t)(lbo >> 4) << 16) + (b_off >> 4);
#pragma unroll
    for (int s = 0; s < KA; ++s) tc::mma_ts(d_tmem, a_tmem + 8 * s, d + ((s * 2 * lbo) >> 4), idesc, s > 0);
    if constexpr (HID) tc::mma_ts(d_tmem, g.bias0 + 8 * bias_chunk, d + ((KA * 2 * lbo) >> 4), idesc, 1);
    tc::mma_commit(bar);
  }
  hook();
}
struct NoOp {
  __device__ void operator()() const {}
};

// Query: the frame layer (N = 16 into F) and the sampler's first layer (N =
// SW into E) both read input chunk 0 — one barrier, one commit.
template <int SW, int LW>
__device__ __forceinline__ void mma_issue_first2(const GG& g, uint32_t f_tmem, uint32_t e_tmem,
                                                 uint32_t a_tmem, uint32_t frame_off, uint32_t s1_off,
                                                 uint64_t* bar) {
  tc::tmem_st_wait();
  tc::tc_fence_before();
  tc::named_bar(g.bar_id, 128);
  if (g.r == 32 * LW) {
    tc::tc_fence_after();
    tc::mma_ts(f_tmem, a_tmem, g.desc0 + ((uint64_t)((16 * 16) >> 4) << 16) + (frame_off >> 4),
               tc::idesc_f16(128, 16), 0);
    tc::mma_ts(e_tmem, a_tmem, g.desc0 + ((uint64_t)((SW * 16) >> 4) << 16) + (s1_off >> 4),
               tc::idesc_f16(128, SW), 0);
    tc::mma_commit(bar);
  }
}

// D[0, W) -> scaled leaky -> (hi, lo) into A, in chunks of NMQ_EPI_COLS
// columns (16 keeps the stage's register peak low; 32 halves the TMEM waits)
#ifndef NMQ_EPI_COLS
#define NMQ_EPI_COLS 16  // measured: 16 > 32 on C2 (30.1 vs 27.8 G q/s with the same kernel otherwise)
#endif
template <int W>
__device__ __forceinline__ void hidden_epi(uint32_t dl, uint32_t al) {
  constexpr int C = W < NMQ_EPI_COLS ? W : NMQ_EPI_COLS;
#pragma unroll
  for (int c0 = 0; c0 < W; c0 += C) {
    uint32_t r[C];
    if constexpr (C == 16) tc::tmem_ld16(dl + c0, r);
    else tc::tmem_ld32(dl + c0, r);
    tc::tmem_ld_wait();
    uint32_t hi[C / 2], lo[C / 2];
#pragma unroll
    for (int j = 0; j < C / 2; ++j) split_scaled(r[2 * j], r[2 * j + 1], hi[j], lo[j]);
    if constexpr (C == 16) {
      tc::tmem_st8(al + c0 / 2, hi);
      tc::tmem_st8(al + W / 2 + c0 / 2, lo);
    } else {
      tc::tmem_st16(al + c0 / 2, hi);
      tc::tmem_st16(al + W / 2 + c0 / 2, lo);
    }
  }
}

// BRDF output layer W -> 3 (6 with albedo) on the CUDA cores from the last
// hidden layer's scaled pre-activations in D: a~ = P + k|P| (FFMA2), then
// y_j = (sum_k w_jk a~_k) / c^depth + b_j.
template <int W>
__device__ __forceinline__ void out_layer_simt(uint32_t dl, const MatParams& mp, float inv_scale,
                                               bool albedo, float (&y)[6]) {
  float2 av[W / 2];
#pragma unroll
  for (int c0 = 0; c0 < W; c0 += 32) {
    constexpr int kChunk = W < 32 ? W : 32;
    uint32_t r[32];
    if constexpr (W == 16) {
      uint32_t r16[16];
      tc::tmem_ld16(dl, r16);
      tc::tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) r[i] = r16[i];
    } else {
      tc::tmem_ld32(dl + c0, r);
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

// Stage one tile's inputs into `ib`: TMA bulk copies for full tiles (issued
// by one thread), direct per-row copies for the partial last tile and for
// gathered rows (a.idx: binned multi-material segments read the caller's
// arrays through the segment's row list instead of a permuted copy).  A
// thread reads only its own row of `ib`, so per-row copies need no barrier.
template <int MODE, bool GATHER>
__device__ __forceinline__ void stage_inputs(const QueryArgs& a, int64_t base, int64_t n, int tile,
                                             InBuf<MODE>& ib, uint64_t* bar, int r, bool issuer) {
  const int64_t q0 = base + (int64_t)tile * kTile;
  if ((!GATHER || !a.idx) && (int64_t)tile * kTile + kTile <= n) {
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
    return;
  }
  const bool v = (int64_t)tile * kTile + r < n;
  if (GATHER && a.idx && v) {  // gathered row: asynchronous 4-byte copies, awaited in wait_in
    const int64_t q = __ldg(a.idx + q0 + r);
    tc::cp_async4(tc::smem_u32(&ib.uv[2 * r]), a.uv + 2 * q);
    tc::cp_async4(tc::smem_u32(&ib.uv[2 * r + 1]), a.uv + 2 * q + 1);
    if (a.lod_stride) tc::cp_async4(tc::smem_u32(&ib.lod[r]), a.lod + q);
    tc::cp_async4(tc::smem_u32(&ib.urr[r]), a.u_rr + q);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      tc::cp_async4(tc::smem_u32(&ib.wi[3 * r + k]), a.wi + 3 * q + k);
      if constexpr (Need<MODE>::wo) tc::cp_async4(tc::smem_u32(&ib.wo[3 * r + k]), a.wo + 3 * q + k);
      if constexpr (Need<MODE>::u3) tc::cp_async4(tc::smem_u32(&ib.u3[3 * r + k]), a.u3 + 3 * q + k);
    }
    tc::cp_async_commit();
    return;
  }
  const int64_t q = q0 + r;
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
}

// Texel prefetch: level + taps of one row and its 4 texel loads (LDG.128,
// L1-cached: the coarse pyramid levels live in L1).  The bilinear weights
// are recomputed in float64 from the row's uv when the texels are blended.
struct TexPrefetch {
  uint4 tex[4];
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
#pragma unroll
  for (int k = 0; k < 4; ++k) p.tex[k] = __ldg(mp.latent + tap_index(t, k));
}

// SMEM variant (TS): the four texels go to this row's 64-byte slot in SMEM
// by cp.async (LDGSTS, L1-allocating) — no registers held across the MLP
// chain; only the level stays live.
template <int MODE>
__device__ __forceinline__ void prefetch_texels_smem(const MatParams& mp, const QueryArgs& a,
                                                     const InBuf<MODE>& ib, int r, float lod0,
                                                     uint32_t row_smem, TexPrefetch& p) {
  const float u = ib.uv[2 * r], v = ib.uv[2 * r + 1];
  const float lod = a.lod_stride ? ib.lod[r] : lod0;
  p.level = choose_level(mp, lod, ib.urr[r]);
  const Taps t = make_taps(mp, p.level, u, v);
#pragma unroll
  for (int k = 0; k < 4; ++k) tc::cp_async16(row_smem + 16 * k, mp.latent + tap_index(t, k));
  tc::cp_async_commit();
}
__device__ __forceinline__ void land_texels_smem(uint32_t row_smem, TexPrefetch& p) {
  tc::cp_async_wait<0>();
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(p.tex[k].x), "=r"(p.tex[k].y), "=r"(p.tex[k].z), "=r"(p.tex[k].w)
                 : "r"(row_smem + 16 * k)
                 : "memory");
}

// Blended latent code of one row as packed fp16 pairs (the MLP input
// rounding): float64 weights and blend, as latent.py:93-97.
template <int MODE>
__device__ __forceinline__ void blend_pack(const MatParams& mp, const TexPrefetch& p, const InBuf<MODE>& ib,
                                           int r, uint32_t (&zp)[4]) {
  const LevelDesc L = mp.lv[p.level];
  double w[4];
  weights64(frac64(ib.uv[2 * r], L.w), frac64(ib.uv[2 * r + 1], L.h), w);
  float z[8];
  blend64<true>(p.tex, w, z);
#pragma unroll
  for (int c = 0; c < 4; ++c) zp[c] = pack2(z[2 * c], z[2 * c + 1]);
}

// Per-slot state (registers; every index is compile-time after unrolling).
struct SlotSt {
  uint32_t d0, a0;  // lane-0 TMEM addresses: accumulator D, input A (frame D at a0 + 16)
  uint32_t dl, al;  // the same with this warp's lane field
  uint32_t e0, el;  // query: sampler layer-1 accumulator (lane 0 / this warp's lanes)
  uint64_t* bar;    // MMA completion barrier
  uint32_t ph;      // its parity
  int t;            // current tile (>= ntiles: idle)
  int it;           // tiles done by this slot (input buffer parity)
  uint32_t ph_bits;  // per input buffer: mbarrier parity of its TMA fills
  uint32_t zp[4];   // fp16 latent code of the current tile's row
  int level;
  V3 wi, u3;        // the row's directions (registers: the buffer is refilled early)
  bool up;          // wi.z > 0 && wo.z > 0
  TexPrefetch nx;   // texels of the slot's next tile
  int32_t qslot;    // spp-mean launches: this row's resolve-queue entry (-1: none)
};

// Follow-up of a BRDF-mode launch: blocks (b, *) resolve the rows CTA b
// queued.  Phase 1, one thread per entry: recompute the row's direction
// inputs in the reference's arithmetic (tw_exact) and compare them with the
// fast ones; rows that differ go to a block list.  Phase 2, one warp per
// listed row: the BRDF decoder on the CUDA cores in fp32 (lane j owns hidden
// units j and j + 32), its fp16 weights read straight from the material's
// UMMA blob (row n's 8-value K chunk c at b_off + c * n_pad * 16 + n * 16:
// one 16-byte load each, all issued up front) and the output layer from the
// fp32 copy in the parameter block.
constexpr int kResolveThreads = 512;
#ifndef NMQ_RESOLVE_FUSED
#define NMQ_RESOLVE_FUSED 1  // resolve in the fast kernel's epilogue (1) or a follow-up kernel (0)
#endif

__device__ __forceinline__ void load_row8(const MatParams& mp, uint32_t off, int n_pad, int n, int c,
                                          float (&w)[8]) {
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(mp.wblob) + off +
                                                       (size_t)c * n_pad * 16 + (size_t)n * 16));
  const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = unpack_h2(u[i]);
    w[2 * i] = f.x;
    w[2 * i + 1] = f.y;
  }
}

template <int BW, int BNH, bool RED = false>
__device__ __forceinline__ void resolve_entries(const MatParams& mp, const QueryArgs& a, const uint4* ent,
                                                uint32_t n, uint32_t first, uint32_t step, uint32_t tid,
                                                uint32_t cap) {
  const int lane = tid & 31;
  const bool seg_out = a.out_idx != nullptr;
  for (uint32_t b0 = first; b0 < n; b0 += step) {  // warp-uniform trip count
    const uint32_t i = b0 + tid;
    uint32_t zh[4] = {0u, 0u, 0u, 0u}, xe[6] = {0u, 0u, 0u, 0u, 0u, 0u};
    int32_t row = 0;
    bool mism = false;
    if (i < n) {
      const uint4* e = ent + i;
      const uint4 e0 = __ldg(e), e1 = __ldg(e + cap), e2 = __ldg(e + 2 * cap), e3 = __ldg(e + 3 * cap),
                  e4 = __ldg(e + 4 * cap);
      row = (int32_t)e0.x;
      zh[0] = e1.w; zh[1] = e2.x; zh[2] = e2.y; zh[3] = e2.z;
      const V3 wi = v3(__uint_as_float(e2.w), __uint_as_float(e3.x), __uint_as_float(e3.y));
      const V3 wo = v3(__uint_as_float(e3.z), __uint_as_float(e3.w), __uint_as_float(e4.x));
      // only this row's frames with a value near a rounding midpoint need the
      // float64 path (tw_resolve runs one frame per lane per pass)
      const uint32_t fm = e4.y;
      tw_resolve(mp, zh, wi, wo, xe, fm);
      const uint32_t xf[6] = {e0.y, e0.z, e0.w, e1.x, e1.y, e1.z};
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const uint32_t own = (fm & 1u ? frame0_halves(c) : 0u) | (fm & 2u ? ~frame0_halves(c) : 0u);
        xe[c] = (xe[c] & own) | (xf[c] & ~own);  // frames not recomputed keep their fast values
        mism |= xe[c] != xf[c];
      }
    }
    // the warp re-evaluates each of its rows whose inputs round differently
    uint32_t mm = __ballot_sync(0xffffffffu, mism);
    while (mm) {
      const int src = __ffs(mm) - 1;
      mm &= mm - 1;
      // BRDF layer 1 on input chunk [z(8) | wi-slot, bias @ 3 | T.wi(6), T.wo(6)]
      // (the pipelined kernels' K order, fill_fast_layers): rows j, j + 32
      float x[20];
#pragma unroll
      for (int c = 0; c < 10; ++c) {
        const float2 f = unpack_h2(__shfl_sync(0xffffffffu, c < 4 ? zh[c & 3] : xe[(c - 4) % 6], src));
        x[2 * c] = f.x;
        x[2 * c + 1] = f.y;
      }
      const int j0 = lane < BW ? lane : 0, j1 = lane + 32 < BW ? lane + 32 : 0;
      float w1[2][4][8];
#pragma unroll
      for (int u = 0; u < (BW > 32 ? 2 : 1); ++u)
#pragma unroll
        for (int c = 0; c < 4; ++c) load_row8(mp, mp.fast_l1_off, BW, u ? j1 : j0, c, w1[u][c]);
      float h[2] = {0.f, 0.f};
#pragma unroll
      for (int u = 0; u < (BW > 32 ? 2 : 1); ++u) {
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __fmaf_rn(x[q], w1[u][0][q], acc);  // z
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = __fmaf_rn(x[8 + q], w1[u][2][q], acc);  // T.wi, T.wo[0..1]
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = __fmaf_rn(x[16 + q], w1[u][3][q], acc);  // T.wo[2..5]
        acc += w1[u][1][3];  // bias
        h[u] = acc >= 0.f ? acc : kLeaky * acc;
      }
#pragma unroll
      for (int l = 1; l < BNH; ++l) {  // hidden layers BW -> BW: K chunks [W (BW/8) | W | bias]
        const LayerDesc& L = mp.layers[mp.brdf_first + l];
        float w[2][BW / 8][8], bb[2][8];
#pragma unroll
        for (int u = 0; u < (BW > 32 ? 2 : 1); ++u) {
#pragma unroll
          for (int c = 0; c < BW / 8; ++c) load_row8(mp, L.b_off, BW, u ? j1 : j0, c, w[u][c]);
          load_row8(mp, L.b_off, BW, u ? j1 : j0, 2 * BW / 8, bb[u]);
        }
        float acc[2] = {0.f, 0.f};
#pragma unroll
        for (int q = 0; q < BW; ++q) {  // every lane takes part in the shuffles
          const float hq = __shfl_sync(0xffffffffu, q < 32 ? h[0] : h[1], q & 31);
#pragma unroll
          for (int u = 0; u < (BW > 32 ? 2 : 1); ++u) acc[u] = __fmaf_rn(hq, w[u][q / 8][q % 8], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < (BW > 32 ? 2 : 1); ++u) {
          const float v = acc[u] + bb[u][0];
          h[u] = v >= 0.f ? v : kLeaky * v;
        }
      }
      if (lane >= BW) h[0] = 0.f;
      // output layer BW -> 3 (6 with albedo), fp32 copy in the parameter block: warp sums
      // (weights from the fp32 copy in global memory: a per-lane index into the
      // constant bank would serialize the warp)
      const LayerDesc& LO = mp.layers[mp.brdf_first + BNH];
      const float* wout = mp.w32 + LO.w32_off;
      float y[6];
#pragma unroll
      for (int o = 0; o < 6; ++o) {
        float p = 0.f;
        if (o < LO.out) {
          p = lane < BW ? h[0] * __ldg(wout + o * (BW + 1) + lane) : 0.f;
          if (BW > 32) p = __fmaf_rn(h[1], __ldg(wout + o * (BW + 1) + 32 + lane), p);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) p += __shfl_xor_sync(0xffffffffu, p, d);
        y[o] = p + mp.ob[o];
      }
      if (RED && lane == src) {  // replace the fast value's share of its pixel's mean
        const uint4 e5 = __ldg(ent + 5 * (size_t)cap + i);
        const float inv = __int_as_float((127 - a.spp_log2) << 23);
        float* o = a.img + 3 * ((int64_t)row >> a.spp_log2);
        atomicAdd(o, (brdf_output(y[0]) - __uint_as_float(e5.x)) * inv);
        atomicAdd(o + 1, (brdf_output(y[1]) - __uint_as_float(e5.y)) * inv);
        atomicAdd(o + 2, (brdf_output(y[2]) - __uint_as_float(e5.z)) * inv);
      } else if (lane == src) {
        const int64_t q = seg_out ? (int64_t)__ldg(a.out_idx + row) : (int64_t)row;
        // queued rows are above the horizon (below it the output is 0 either way)
        stg3(a.rgb, q, v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2])));
        if (mp.albedo && a.albedo) stg3(a.albedo, q, v3(fmaxf(y[3], 0.f), fmaxf(y[4], 0.f), fmaxf(y[5], 0.f)));
      }
    }
  }
}

template <int BW, int BNH>
__global__ void __launch_bounds__(kResolveThreads, 2)
resolve_kernel(const __grid_constant__ MatParams mp, const __grid_constant__ QueryArgs a,
               const __grid_constant__ FastConsts fc) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the fast kernel's queue and outputs
  resolve_entries<BW, BNH>(mp, a, fc.q.ent + kQueueWords * (size_t)blockIdx.x * fc.q.cap, fc.q.cnt[blockIdx.x],
                           blockIdx.y * kResolveThreads, kResolveThreads * gridDim.y, threadIdx.x, fc.q.cap);
}

template <int MODE, int BW, int BNH, int SW, int SNH, int G, int NS, bool TS, bool SEG, bool DBG = false,
          bool RED = false>
__global__ void __launch_bounds__(G * 128, 1)
fast_kernel(const __grid_constant__ MatParams mp, const __grid_constant__ QueryArgs a,
            const __grid_constant__ FastConsts fc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mma_bar[G][NS];  // MMA completion
  __shared__ uint64_t in_bar[G][NS][2];
  __shared__ uint64_t w_bar;  // weights staged by TMA
  __shared__ uint32_t tbase_sh;
  __shared__ uint32_t q_cnt;  // BRDF modes: rows this CTA queued for exact resolution
  constexpr bool kBrdf = Need<MODE>::brdf, kSamp = Need<MODE>::samp;
  // stage layout of one tile (see the file comment)
  // query: the sampler's first layer reads the same input chunk 0 as the
  // frame layer, so both are issued together (its D in a third region E) and
  // the sampler chain starts at the BRDF output stage: one round trip less
  constexpr bool kQM = kBrdf && kSamp;
  constexpr int kOutB = kBrdf ? BNH : -1;                   // BRDF output stage
  constexpr int kS0 = kBrdf ? (kQM ? BNH : BNH + 1) : 0;    // stage issuing sampler layer 2
  constexpr int kFinal = kSamp ? kS0 + SNH : kOutB;         // last stage
  constexpr int kStages = kFinal + 1;
  constexpr int DW = BW > SW ? BW : SW;
  static_assert(DW >= 32, "frame-layer D aliases A columns [16, 32)");
  constexpr uint32_t kSlotCols = 2 * DW + (kQM ? SW : 0);
  constexpr uint32_t kBiasCol = G * NS * kSlotCols;
  constexpr uint32_t kUsedCols = kBiasCol + 32;
  static_assert(kUsedCols <= 512, "TMEM budget");
  // power-of-two allocation covering all slots + bias chunks, so CTAs that
  // happen to share an SM never block each other in tcgen05.alloc
  constexpr uint32_t kTmemCols = kUsedCols <= 128 ? 128 : (kUsedCols <= 256 ? 256 : 512);

  const int tid = threadIdx.x;
  // warp-uniform by construction (shfl from lane 0): lets ptxas keep the
  // TMEM/MMA operands in uniform registers (no R2UR waterfall per MMA)
  const int gi = __shfl_sync(0xffffffffu, tid / 128, 0), r = tid % 128;
  const int warp = tid / 32;

  const uint32_t wbytes = (mp.wblob_bytes + 127) & ~127u;
  InBuf<MODE>* ibuf = reinterpret_cast<InBuf<MODE>*>(smem + wbytes) + gi * NS * 2;
  // TS: per-row 64-byte texel slots after all input buffers
  const uint32_t tex_row = tc::smem_u32(smem + wbytes + G * NS * 2 * sizeof(InBuf<MODE>)) +
                           (uint32_t)((gi * NS) * kTile + tid % 128) * 64u;

  // --- CTA setup --------------------------------------------------------------
  if (tid == 0) q_cnt = 0u;
  if (tid < G * NS) {
    tc::mbar_init(&mma_bar[tid / NS][tid % NS], 1);
    tc::mbar_init(&in_bar[tid / NS][tid % NS][0], 1);
    tc::mbar_init(&in_bar[tid / NS][tid % NS][1], 1);
  }
  if (tid == 32) {
    // weights: 1-D TMA bulk copies (multiples of 16 B), overlapped with the
    // prologue's input staging and texel fetch
    tc::mbar_init(&w_bar, 1);
    tc::fence_mbar_init();
    tc::mbar_arrive_expect_tx(&w_bar, mp.wblob_bytes);
    for (uint32_t o = 0; o < mp.wblob_bytes; o += 32768u) {
      const uint32_t nb = mp.wblob_bytes - o < 32768u ? mp.wblob_bytes - o : 32768u;
      tc::tma_load_1d(tc::smem_u32(smem + o), reinterpret_cast<const uint8_t*>(mp.wblob) + o, nb,
                      &w_bar);
    }
  }
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&tbase_sh);
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

  GG g;
  g.bias0 = tb + kBiasCol;
  g.desc0 = tc::smem_desc(tc::smem_u32(smem), 0, 128);
  g.bar_id = 1 + gi;
  g.r = r;
  static_assert(1 + G <= 16, "named barriers");
  const uint32_t lane = (uint32_t)((warp & 3) * 32) << 16;

  // programmatic dependent launch: everything above (barriers, TMEM, the
  // material's weights) is independent of earlier work on the stream; wait
  // for it here, before the first read of the inputs or write of the outputs
  if constexpr (NMQ_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
  const float lod0 = a.lod_stride ? 0.f : __ldg(a.lod);
  // SEG: a binned segment (device row range + output-row indirection); the
  // plain instantiation carries none of it
  const int64_t seg_base = SEG && a.seg ? (int64_t)__ldg(a.seg) : 0;
  const int64_t n_rows = SEG && a.seg ? (int64_t)__ldg(a.seg + 1) : a.n;
  const bool seg_out = SEG && a.out_idx;
  const int ntiles = (int)((n_rows + kTile - 1) / kTile);  // host guarantees < 2^31
  const int last_full = SEG && a.idx ? 0 : (int)(n_rows / kTile);  // tiles [0, last_full) staged by TMA
  const int stride = gridDim.x * G;                        // between a group's tiles
  const int sstride = stride * NS;                         // between a slot's tiles
  const bool want_level = a.level != nullptr;
  const bool want_albedo = mp.albedo && a.albedo;

  SlotSt sl[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    sl[s].d0 = tb + (gi * NS + s) * kSlotCols;
    sl[s].a0 = sl[s].d0 + DW;
    sl[s].dl = sl[s].d0 + lane;
    sl[s].al = sl[s].a0 + lane;
    sl[s].e0 = sl[s].a0 + DW;
    sl[s].el = sl[s].e0 + lane;
    sl[s].bar = &mma_bar[gi][s];
    sl[s].ph = 0u;
    sl[s].t = blockIdx.x * G + gi + s * stride;
    sl[s].it = 0;
    sl[s].ph_bits = 0u;
  }
  auto buf = [&](int s, int b) -> InBuf<MODE>& { return ibuf[s * 2 + b]; };
  // inputs of `tile` in buffer b: full tiles arrive by TMA, the partial last
  // tile was copied row by row by its own threads (no wait needed)
  auto wait_in = [&](SlotSt& S, int s, int b, int tile) {
    if (tile < last_full) {
      tc::mbar_wait(&in_bar[gi][s][b], (S.ph_bits >> b) & 1u);
      S.ph_bits ^= 1u << b;
    } else if (SEG && a.idx) {
      tc::cp_async_wait<0>();  // this thread's gathered row (and any older copies)
    }
  };
  // First MMA of a tile: input chunk 0 = [z, wi, 1] -> frame layer (eval /
  // query; D at A + 16) or sampler layer 1 (sample+pdf).
  auto issue_first = [&](SlotSt& S, const InBuf<MODE>& ib, auto lwc) {
    constexpr int LW = decltype(lwc)::value;
    const uint32_t x[8] = {S.zp[0], S.zp[1], S.zp[2], S.zp[3],
                           pack2(ib.wi[3 * r], ib.wi[3 * r + 1]), pack2(ib.wi[3 * r + 2], 1.f), 0u, 0u};
    tc::tmem_st8(S.al, x);
    if constexpr (kQM)
      mma_issue_first2<SW, LW>(g, S.a0 + 16, S.e0, S.a0, mp.fast_frame_off, mp.layers[mp.samp_first].b_off,
                               S.bar);
    else if constexpr (kBrdf)
      mma_issue<16, 1, false, LW>(g, S.a0 + 16, S.a0, mp.fast_frame_off, 0, S.bar, NoOp{});
    else
      mma_issue<SW, 1, false, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first].b_off, 0, S.bar, NoOp{});
  };

  // --- prologue: per slot stage tiles 0 and 1, fetch + blend tile 0, issue its first MMA
  sfor<NS>([&](auto sc) {
    constexpr int s = decltype(sc)::value;
    SlotSt& S = sl[s];
    if (S.t < ntiles) {
      stage_inputs<MODE, SEG>(a, seg_base, n_rows, S.t, buf(s, 0), &in_bar[gi][s][0], r, r == 64);
      if (S.t + sstride < ntiles)
        stage_inputs<MODE, SEG>(a, seg_base, n_rows, S.t + sstride, buf(s, 1), &in_bar[gi][s][1], r, r == 64);
      wait_in(S, s, 0, S.t);
      TexPrefetch p0;
      prefetch_texels<MODE>(mp, a, buf(s, 0), r, lod0, p0);
      blend_pack<MODE>(mp, p0, buf(s, 0), r, S.zp);
      S.level = p0.level;
      if (s == 0) tc::mbar_wait(&w_bar, 0);  // weights in SMEM before the first MMA
      issue_first(S, buf(s, 0), std::integral_constant<int, s % 4>{});
    }
  });

  // --- main loop: one tile per slot per iteration ----------------------------------
  while (sl[0].t < ntiles) {
    sfor<kStages>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      sfor<NS>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        constexpr int LW = (k + s + 1) % 4;  // issuing warp rotates over the group
        SlotSt& S = sl[s];
        if (s > 0 && S.t >= ntiles) return;  // uniform per group
        const int b = S.it & 1;
        const int64_t q_in = (int64_t)S.t * kTile + r;  // input row
        const bool valid = q_in < n_rows;
        const int t2 = S.t + 2 * sstride;

        if constexpr (k == 0) {
          // this tile's directions -> registers; its input buffer is refilled
          // (tile t2) after the stage's barrier
          const InBuf<MODE>& ib = buf(s, b);
          S.wi = v3(ib.wi[3 * r], ib.wi[3 * r + 1], ib.wi[3 * r + 2]);
          V3 wo = v3(0.f, 0.f, 1.f);
          if constexpr (Need<MODE>::wo) wo = v3(ib.wo[3 * r], ib.wo[3 * r + 1], ib.wo[3 * r + 2]);
          if constexpr (Need<MODE>::u3) S.u3 = v3(ib.u3[3 * r], ib.u3[3 * r + 1], ib.u3[3 * r + 2]);
          S.up = (S.wi.z > 0.f) && (wo.z > 0.f);
          if (want_level) {
            if (valid) a.level[seg_out ? (int64_t)__ldg(a.out_idx + seg_base + q_in) : q_in] = S.level;
          }
          // the slot's next tile: texel loads now, blended at the last stage
          if (S.t + sstride < ntiles) {
            wait_in(S, s, b ^ 1, S.t + sstride);
            if constexpr (TS)
              prefetch_texels_smem<MODE>(mp, a, buf(s, b ^ 1), r, lod0, tex_row + s * kTile * 64u, S.nx);
            else
              prefetch_texels<MODE>(mp, a, buf(s, b ^ 1), r, lod0, S.nx);
          }
          auto refill = [&]() {  // after the barrier: every row of buffer b was read
            if (t2 < last_full) {
              if (r == 32 * ((LW + 2) % 4))
                stage_inputs<MODE, SEG>(a, seg_base, n_rows, t2, buf(s, b), &in_bar[gi][s][b], r, true);
            } else if (t2 < ntiles) {
              stage_inputs<MODE, SEG>(a, seg_base, n_rows, t2, buf(s, b), &in_bar[gi][s][b], r, false);  // own row
            }
          };
          mma_wait(S.bar, S.ph);
          if constexpr (kBrdf) {
            // frame layer D -> frames, T.wi, T.wo -> input chunk 1 -> BRDF layer 1
            uint32_t fr[16];
            tc::tmem_ld16(S.al + 16, fr);
            tc::tmem_ld_wait();
            float raw[12];
#pragma unroll
            for (int j = 0; j < 12; ++j) raw[j] = __uint_as_float(fr[j]);
#if NMQ_TW_INLINE
            {
              (void)raw;
              uint32_t x6[6];
              tw_resolve(mp, S.zp, S.wi, wo, x6, 3u);
              const uint32_t x[8] = {x6[0], x6[1], x6[2], x6[3], x6[4], x6[5], 0u, 0u};
              tc::tmem_st8(S.al + 8, x);
              if constexpr (RED) S.qslot = -1;
              mma_issue<BW, 2, false, LW>(g, S.d0, S.a0, mp.fast_l1_off, 0, S.bar, refill);
            }
            if (false) {
#else
            {
#endif
            float ti[6], to[6];
            const float2 kappa = frames2_transform(raw, S.wi, wo, ti, to);
            const uint32_t x[8] = {pack2(ti[0], ti[1]), pack2(ti[2], ti[3]), pack2(ti[4], ti[5]),
                                   pack2(to[0], to[1]), pack2(to[2], to[3]), pack2(to[4], to[5]),
                                   0u, 0u};
            tc::tmem_st8(S.al + 8, x);
            // exact rounding: a direction input within its error bound of an
            // fp16 midpoint (bound = tw_delta x conditioning of its frame)
            const float2 d1 = make_float2(fc.tw_delta * kappa.x, fc.tw_delta * kappa.x);
            const float2 d2 = make_float2(fc.tw_delta * kappa.y, fc.tw_delta * kappa.y);
            const float2 d12 = make_float2(d1.x, d2.x);
            const uint32_t nw1 = near_mid2(ti[2], ti[3], d12), nw4 = near_mid2(to[2], to[3], d12);
            const uint32_t near_f0 = near_mid2(ti[0], ti[1], d1) | near_mid2(to[0], to[1], d1) |
                                     ((nw1 | nw4) & 0xFFFFu);
            const uint32_t near_f1 = near_mid2(ti[4], ti[5], d2) | near_mid2(to[4], to[5], d2) |
                                     ((nw1 | nw4) >> 16);
            const bool flag = valid && S.up && (near_f0 | near_f1) != 0u;
            // queue the tile's flagged rows (one shared atomic per warp)
            const uint32_t wmask = __ballot_sync(0xffffffffu, flag);
            if constexpr (RED) S.qslot = -1;
            if (wmask) {
              const int lead = __ffs(wmask) - 1;
              uint32_t wbase = 0;
              if ((r & 31) == lead) wbase = atomicAdd(&q_cnt, __popc(wmask));
              wbase = __shfl_sync(0xffffffffu, wbase, lead);
              if (flag) {
                const uint32_t slot = wbase + __popc(wmask & lanemask_lt());
                if constexpr (RED) S.qslot = (int32_t)slot;
                const size_t cap = fc.q.cap;
                uint4* e = fc.q.ent + kQueueWords * (size_t)blockIdx.x * cap + slot;
                e[0] = make_uint4((uint32_t)(seg_base + q_in), x[0], x[1], x[2]);
                e[cap] = make_uint4(x[3], x[4], x[5], S.zp[0]);
                e[2 * cap] = make_uint4(S.zp[1], S.zp[2], S.zp[3], __float_as_uint(S.wi.x));
                e[3 * cap] = make_uint4(__float_as_uint(S.wi.y), __float_as_uint(S.wi.z), __float_as_uint(wo.x),
                                        __float_as_uint(wo.y));
                e[4 * cap] = make_uint4(__float_as_uint(wo.z), (near_f0 ? 1u : 0u) | (near_f1 ? 2u : 0u), 0u, 0u);
              }
            }
            mma_issue<BW, 2, false, LW>(g, S.d0, S.a0, mp.fast_l1_off, 0, S.bar, refill);
            if (DBG && valid) {  // calibration dump (tools/tw_calibrate.py)
              float* o = a.dbg + 14 * (seg_base + q_in);
#pragma unroll
              for (int j = 0; j < 6; ++j) { o[j] = ti[j]; o[6 + j] = to[j]; }
              o[12] = kappa.x;
              o[13] = kappa.y;
            }
            }
          } else {
            // sample+pdf: sampler layer 1 D -> layer 2
            hidden_epi<SW>(S.dl, S.al);
            if constexpr (SNH == 1)
              mma_issue<16, 2 * SW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first + 1].b_off, 1,
                                                   S.bar, refill);
            else
              mma_issue<SW, 2 * SW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first + 1].b_off, 1,
                                                   S.bar, refill);
          }
        } else if constexpr (kBrdf && k < kOutB) {
          // BRDF hidden layer k+1
          mma_wait(S.bar, S.ph);
          hidden_epi<BW>(S.dl, S.al);
          mma_issue<BW, 2 * BW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.brdf_first + k].b_off, k, S.bar,
                                               NoOp{});
        } else if constexpr (k == kOutB) {
          // BRDF output layer on the CUDA cores
          mma_wait(S.bar, S.ph);
          float y[6];
          out_layer_simt<BW>(S.dl, mp, fc.inv_brdf, mp.albedo != 0, y);
          if constexpr (RED) {
            // per-pixel spp mean straight from the epilogue: per-sample rgb
            // never reaches HBM; a queued row keeps its fast value in its entry
            const V3 f = S.up ? v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2])) : v3(0.f, 0.f, 0.f);
            spp_accumulate(a.img, q_in, f, valid, a.spp_log2);
            if (S.qslot >= 0)
              fc.q.ent[kQueueWords * (size_t)blockIdx.x * fc.q.cap + 5 * (size_t)fc.q.cap + S.qslot] =
                  make_uint4(__float_as_uint(f.x), __float_as_uint(f.y), __float_as_uint(f.z), 0u);
          } else if (valid) {
            const int64_t q = seg_out ? (int64_t)__ldg(a.out_idx + seg_base + q_in) : q_in;
            const V3 f = S.up ? v3(brdf_output(y[0]), brdf_output(y[1]), brdf_output(y[2]))
                              : v3(0.f, 0.f, 0.f);
            stg3(a.rgb, q, f);
            if (want_albedo) {
              const V3 al = S.up ? v3(fmaxf(y[3], 0.f), fmaxf(y[4], 0.f), fmaxf(y[5], 0.f))
                                 : v3(0.f, 0.f, 0.f);
              stg3(a.albedo, q, al);
            }
          }
          if constexpr (kQM) {
            // query: sampler layer 1 (issued with the frame layer, in E) -> layer 2
            hidden_epi<SW>(S.el, S.al);
            if constexpr (SNH == 1)
              mma_issue<16, 2 * SW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first + 1].b_off, 1,
                                                   S.bar, NoOp{});
            else
              mma_issue<SW, 2 * SW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first + 1].b_off, 1,
                                                   S.bar, NoOp{});
          }
        } else if constexpr (kSamp && k > kS0 && k < kFinal) {
          // sampler layer j+1 (j = k - kS0 >= 1; stage kS0 is k == 0 or handled above)
          constexpr int j = k - kS0;
          mma_wait(S.bar, S.ph);
          hidden_epi<SW>(S.dl, S.al);
          if constexpr (j + 1 == SNH)
            mma_issue<16, 2 * SW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first + j + 1].b_off, j + 1,
                                                 S.bar, NoOp{});
          else
            mma_issue<SW, 2 * SW / 16, true, LW>(g, S.d0, S.a0, mp.layers[mp.samp_first + j + 1].b_off, j + 1,
                                                 S.bar, NoOp{});
        }
        if constexpr (kSamp && k == kFinal) {
          // proxy parameters, sample, pdf
          mma_wait(S.bar, S.ph);
          uint32_t yr[16];
          tc::tmem_ld16(S.dl, yr);
          tc::tmem_ld_wait();
          float raw[9];
#pragma unroll
          for (int j = 0; j < 9; ++j) raw[j] = __uint_as_float(yr[j]);
          const Proxy p = proxy_from_raw(raw, mp.isotropic != 0, fc.inv_samp);
          if (valid) {
            const int64_t q = seg_out ? (int64_t)__ldg(a.out_idx + seg_base + q_in) : q_in;
            if (a.params9) store_proxy(a.params9, q, p);
            const V3 w = proxy_sample(p, S.wi, S.u3.x, S.u3.y, S.u3.z);
            stg3(a.ws, q, w);
            a.pdf[q] = proxy_pdf(p, S.wi, w);
          }
        }
        if constexpr (k == kFinal) {
          // the slot's next tile: blend its texels, issue its first MMA
          const int tn = S.t + sstride;
          if (tn < ntiles) {
            if constexpr (TS) land_texels_smem(tex_row + s * kTile * 64u, S.nx);
            blend_pack<MODE>(mp, S.nx, buf(s, b ^ 1), r, S.zp);
            S.level = S.nx.level;
            issue_first(S, buf(s, b ^ 1), std::integral_constant<int, LW>{});
          }
          S.t = tn;
          S.it += 1;
        }
      });
    });
  }
  if constexpr (NMQ_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 0) tc::tmem_free<kTmemCols>(tb);
  if constexpr (kBrdf) {
    if (NMQ_RESOLVE_FUSED) {
      // every queued row's output is stored (the barrier above): the CTA
      // resolves its own rows while other SMs are still on their tiles
      resolve_entries<BW, BNH, RED>(mp, a, fc.q.ent + kQueueWords * (size_t)blockIdx.x * fc.q.cap, q_cnt, 0,
                                    G * 128, tid, fc.q.cap);
    } else if (tid == 0) {
      fc.q.cnt[blockIdx.x] = q_cnt;
    }
  }
}

uint32_t fp16_bits(double v) {
  const __half h = __double2half(v);
  return *reinterpret_cast<const uint16_t*>(&h);
}

#ifndef NMQ_TW_DELTA
// error bound of the fast fp32 T.w per unit frame conditioning: measured
// max |fast - exact| / kappa = 1.48e-7 and 1.66e-7 over 6.2M C2 queries x 12
// values each, two builds (tools/tw_calibrate.py, profiles/r02_tw_calibration*.txt);
// ~2x margin.  Refining the MUFU rsqrt by a Newton step did not lower it
// (the tensor-core frame layer's rounding dominates).
#define NMQ_TW_DELTA 3e-7f
#endif

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
  c.tw_delta = g_tw_margin > 0.f ? g_tw_margin : NMQ_TW_DELTA;
  return c;
}

int g_sms = 0;

}  // namespace

float g_tw_margin = 0.f;

namespace {

#ifndef NMQ_TEX_SMEM
// bit per mode (1 << MODE): stage texel prefetches in SMEM by cp.async
// instead of registers — frees ~19 registers/thread; pays off only where it
// buys a tile group (sample+pdf: G 5 -> 6, +3 % on C3; eval/query: no gain)
#define NMQ_TEX_SMEM (1 << kModeSamplePdf)
#endif

// Exact-rounding queue storage: one grow-only buffer per (device, stream) —
// launches on one stream are ordered, so consecutive launches reuse it;
// concurrent streams never share one.  Growth is stream-ordered
// (cudaMallocAsync / cudaFreeAsync on the launch stream).
struct QueueBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
std::mutex g_qmu;
std::map<std::pair<int, cudaStream_t>, QueueBuf> g_queues;

cudaError_t queue_for(cudaStream_t s, size_t bytes, void** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_qmu);
  QueueBuf& q = g_queues[{dev, s}];
  if (q.bytes < bytes) {
    if (q.p) {
      const cudaError_t e = cudaFreeAsync(q.p, s);
      if (e != cudaSuccess) return e;
      q.p = nullptr;
      q.bytes = 0;
    }
    const size_t want = bytes + bytes / 4;
    const cudaError_t e = cudaMallocAsync(&q.p, want, s);
    if (e != cudaSuccess) return e;
    q.bytes = want;
  }
  *out = q.p;
  return cudaSuccess;
}

// non-segment launches larger than this run as several (fast, resolve)
// pairs, which bounds the queue at kChunkRows entries per stream
constexpr int64_t kChunkRows = int64_t(1) << 24;
constexpr unsigned kResolveSlices = 2;  // resolve blocks per fast-kernel CTA

template <class K>
cudaError_t launch_pdl(K kern, dim3 grid, dim3 block, size_t smem, cudaStream_t s, const MatParams& mp,
                       const QueryArgs& a, const FastConsts& fc) {
  if constexpr (NMQ_PDL) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, mp, a, fc);
  } else {
    kern<<<grid, block, smem, s>>>(mp, a, fc);
    return cudaGetLastError();
  }
}

template <int MODE, int BW, int BNH, int SW, int SNH, int G, int NS,
          bool TS = ((NMQ_TEX_SMEM >> MODE) & 1) != 0>
cudaError_t launch_fast_t(const MatParams& mp, const QueryArgs& a, cudaStream_t s) {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool seg = a.seg || a.out_idx || a.idx;  // segment instantiation (gathers rows when a.idx)
  constexpr bool kBrdf = Need<MODE>::brdf;
  if (kBrdf && !seg && a.n > kChunkRows) {
    for (int64_t c0 = 0; c0 < a.n; c0 += kChunkRows) {
      QueryArgs c = a;
      c.n = a.n - c0 < kChunkRows ? a.n - c0 : kChunkRows;
      c.uv = a.uv + 2 * c0;
      c.lod = a.lod_stride ? a.lod + c0 : a.lod;
      c.u_rr = a.u_rr + c0;
      c.wi = a.wi + 3 * c0;
      if (a.wo) c.wo = a.wo + 3 * c0;
      if (a.u3) c.u3 = a.u3 + 3 * c0;
      if (a.rgb) c.rgb = a.rgb + 3 * c0;
      if (a.albedo) c.albedo = a.albedo + 3 * c0;
      if (a.ws) c.ws = a.ws + 3 * c0;
      if (a.pdf) c.pdf = a.pdf + c0;
      if (a.params9) c.params9 = a.params9 + 9 * c0;
      if (a.level) c.level = a.level + c0;
      if (a.dbg) c.dbg = a.dbg + 14 * c0;
      if (a.img) c.img = a.img + 3 * (c0 >> a.spp_log2);  // chunks are whole pixels (2^24 rows)
      const cudaError_t e = launch_fast_t<MODE, BW, BNH, SW, SNH, G, NS, TS>(mp, c, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (a.img && (MODE != kModeEval || seg || !NMQ_RESOLVE_FUSED)) return cudaErrorNotSupported;
  auto kern = seg ? fast_kernel<MODE, BW, BNH, SW, SNH, G, NS, TS, true>
              : (a.dbg && MODE == kModeEval) ? fast_kernel<MODE, BW, BNH, SW, SNH, G, NS, TS, false, true>
              : (a.img && MODE == kModeEval) ? fast_kernel<MODE, BW, BNH, SW, SNH, G, NS, TS, false, false, true>
                                             : fast_kernel<MODE, BW, BNH, SW, SNH, G, NS, TS, false>;
  const int smem = (int)(((mp.wblob_bytes + 127) & ~127u) + G * NS * 2 * sizeof(InBuf<MODE>) +
                         (TS ? G * NS * kTile * 64 : 0));
  const int max_dyn = std::min(max_dynamic_smem((const void*)fast_kernel<MODE, BW, BNH, SW, SNH, G, NS, TS, false>),
                               max_dynamic_smem((const void*)kern));
  if (max_dyn < 0) return cudaErrorInvalidValue;
  if (smem > max_dyn) return cudaErrorNotSupported;
  const int64_t ntiles = (a.n + kTile - 1) / kTile;
  int64_t grid = g_sms;
  if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
  if (grid > (ntiles + G - 1) / G) grid = (ntiles + G - 1) / G;
  if (grid < 1) grid = 1;
  FastConsts fc = make_consts(BNH, SNH);
  if constexpr (kBrdf) {
    // a CTA runs at most G * NS * ceil(ntiles / (grid * G * NS)) tiles
    const int64_t per = (int64_t)G * NS * ((ntiles + grid * G * NS - 1) / (grid * G * NS)) * kTile;
    void* qb = nullptr;
    const size_t ent_bytes = (size_t)grid * per * 16 * kQueueWords;
    cudaError_t e = queue_for(s, ent_bytes + (size_t)grid * 4, &qb);
    if (e != cudaSuccess) return e;
    fc.q.ent = reinterpret_cast<uint4*>(qb);
    fc.q.cnt = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(qb) + ent_bytes);
    fc.q.cap = (uint32_t)per;
  }
  cudaError_t e = launch_pdl(kern, dim3((unsigned)grid), dim3(G * 128), (size_t)smem, s, mp, a, fc);
  if (e != cudaSuccess) return e;
  ++g_launches;
  if constexpr (kBrdf) if (!NMQ_RESOLVE_FUSED) {
    e = launch_pdl(resolve_kernel<BW, BNH>, dim3((unsigned)grid, kResolveSlices), dim3(kResolveThreads), 0, s,
                   mp, a, fc);
    if (e != cudaSuccess) return e;
    ++g_launches;
  }
  return cudaGetLastError();
}

template <int BW, int BNH, int SW, int SNH, int GE, int GS, int GQ, int NS>
cudaError_t launch_fast_arch(int mode, const MatParams& mp, const QueryArgs& a, cudaStream_t s) {
  switch (mode) {
    case kModeEval: return launch_fast_t<kModeEval, BW, BNH, SW, SNH, GE, NS>(mp, a, s);
    case kModeSamplePdf: return launch_fast_t<kModeSamplePdf, BW, BNH, SW, SNH, GS, NS>(mp, a, s);
    case kModeQuery: return launch_fast_t<kModeQuery, BW, BNH, SW, SNH, GQ, NS>(mp, a, s);
    default: return cudaErrorNotSupported;
  }
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

// Returns cudaErrorNotSupported when the fast path does not apply (caller
// then uses the generic kernel).
cudaError_t launch_fast(const MatParams& mp, int mode, const QueryArgs& a, cudaStream_t s) {
  if (mp.fast_arch < 0 || mp.texel_fp32 || a.uv64 || a.wi64) return cudaErrorNotSupported;
  if (mode != kModeEval && mode != kModeSamplePdf && mode != kModeQuery)
    return cudaErrorNotSupported;
  if (!aligned16(a.uv) || !aligned16(a.u_rr) || !aligned16(a.wi) ||
      (a.lod_stride && !aligned16(a.lod)) || (a.wo && !aligned16(a.wo)) ||
      (a.u3 && !aligned16(a.u3)))
    return cudaErrorNotSupported;
  switch (mp.fast_arch) {
    case 0:
      return launch_fast_arch<32, 2, 32, 3, NMQ_G_EVAL, NMQ_G_SAMPLE, NMQ_G_QUERY, NMQ_FAST_NS>(mode, mp, a, s);
    case 1:
      return launch_fast_arch<16, 2, 32, 3, NMQ_G_EVAL, NMQ_G_SAMPLE, NMQ_G_QUERY, NMQ_FAST_NS>(mode, mp, a, s);
    case 2: return launch_fast_arch<64, 3, 32, 3, 3, 3, 3, 1>(mode, mp, a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace nmq
