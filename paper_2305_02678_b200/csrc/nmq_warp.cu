// nmq_warp.cu — warp-tile fused query kernels (the coherent per-material
// path).  Each warp owns a 32-query tile end to end: no block
// barriers, no cross-warp hand-offs, no accumulator round trips through
// memory.  The MLP layers run on the tensor cores with warp-level
// mma.sync.m16n8k16 / m16n8k8 (fp16 x fp16 -> fp32): the 32 queries are two
// 16-row tiles, a layer's fp32 accumulator fragment is re-packed in
// registers into the next layer's A fragment (the C->A layout identity), and
// the per-query nonlinear steps (latent fetch, shading frames, proxy, sample,
// pdf) run one query per lane.  Row <-> fragment transposes go through a
// 2 KB per-warp SMEM stage (stmatrix-free: 16-byte stores + ldmatrix).
//
// Design alternative to the pipelined tcgen05 kernel (nmq_fast.cu), kept as
// kernel path 3: no block barriers and ~20-cycle MMA latency, but 4x lower
// tensor throughput (1024 MAC/clk/SM measured, tools/hmmaprobe.cu) against
// ~3.8k padded MACs per eval query (hi/lo doubles every hidden layer), and
// ~125 registers per thread (16 warps/SM).  Measured on B200 (C2 eval):
// 22.8 G queries/s vs 31.4 G for the tcgen05 kernel, which stays the default.
//
// Exactness as in nmq_fast.cu: inputs rounded to fp16 once (the reference's
// fused_forward), every hidden activation split a~ = hi + lo (fp16 each,
// scaled-leaky a~ = y + k|y|), both halves multiplied by the same fp16
// weight fragment; biases enter as fp32 accumulator init (times c^depth).
#include <cstdint>
#include <cmath>
#include <cuda_fp16.h>
#include <utility>
#include "tc.cuh"
#include "nmq_device.cuh"
#include "nmq_internal.h"

namespace nmq {
namespace {

using namespace dev;

#ifndef NMQ_WARPS
#define NMQ_WARPS 16  // warps per CTA (one CTA per SM)
#endif

constexpr int kWT = 32;  // queries per warp tile
constexpr float kLk = 0.98019802570343017578f;  // fp32(99/101), see nmq_fast.cu

template <int MODE>
struct WNeed {
  static constexpr bool wo = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool u3 = (MODE == kModeSamplePdf || MODE == kModeQuery);
  static constexpr bool brdf = (MODE == kModeEval || MODE == kModeQuery);
  static constexpr bool samp = (MODE == kModeSamplePdf || MODE == kModeQuery);
};

// one warp tile's inputs in SMEM (1-D TMA bulk copies, 16-byte multiples)
template <int MODE>
struct alignas(16) WIn {
  float uv[2 * kWT];
  float lod[kWT];
  float urr[kWT];
  float wi[3 * kWT];
  float wo[WNeed<MODE>::wo ? 3 * kWT : 4];
  float u3[WNeed<MODE>::u3 ? 3 * kWT : 4];
};

template <int... I, class F>
__device__ __forceinline__ void sfor_impl(std::integer_sequence<int, I...>, F&& f) {
  (f(std::integral_constant<int, I>{}), ...);
}
template <int N, class F>
__device__ __forceinline__ void sfor(F&& f) {
  sfor_impl(std::make_integer_sequence<int, N>{}, f);
}

// ---- warp-level MMA and ldmatrix ------------------------------------------------
// m16n8k16: A rows (g, g+8) x k (2t.., 2t+8..); B k x n(g); C/D rows (g, g+8) x cols (2t, 2t+1)
__device__ __forceinline__ void mma16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0));
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void ldsm2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(addr)
               : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
__device__ __forceinline__ void sts64f(uint32_t addr, float a, float b) {
  asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ float2 lds64f(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr) : "memory");
  return v;
}

// Per-warp stage: 32 rows x 64 bytes, 16-byte chunk c of row r stored at
// chunk c ^ ((r >> 1) & 3) (conflict-free ldmatrix / row-wise LDS.128).
__device__ __forceinline__ uint32_t stg(uint32_t base, int row, int chunk) {
  return base + row * 64 + ((chunk ^ ((row >> 1) & 3)) << 4);
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void split_scaled(float ya, float yb, uint32_t& hi, uint32_t& lo) {
  // a~ = y + k|y| for the pair (one FFMA2 with |.|), then fp16 (hi, lo), hi + lo = a~ to ~2^-22
  const float2 ab = __ffma2_rn(make_float2(fabsf(ya), fabsf(yb)), make_float2(kLk, kLk),
                               make_float2(ya, yb));
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

// B fragments of one layer (K = 16*KS, N = 8*NT) from the SMEM weight blob:
// b[nt][ks][0..1]; chunk c of row n at off + c*npad*16 + n*16.
template <int NT, int KS>
struct BFrag {
  uint32_t b[NT][KS][2];
};
template <int NT, int KS>
__device__ __forceinline__ void load_b(uint32_t wbase, uint32_t off, int lane, BFrag<NT, KS>& f) {
  constexpr int npad = NT * 8;  // the host packs every layer with n_pad = 8 * n-tiles
  if constexpr (NT == 1) {
    if constexpr (KS == 1) {
      ldsm2(wbase + off + ((lane >> 3) & 1) * npad * 16 + (lane & 7) * 16, f.b[0][0][0], f.b[0][0][1]);
    } else {
      static_assert(KS % 2 == 0, "");
#pragma unroll
      for (int ks = 0; ks < KS; ks += 2) {  // x4 = chunks 2ks .. 2ks+3 of rows 0-7
        uint32_t r[4];
        ldsm4(wbase + off + (2 * ks + (lane >> 3)) * npad * 16 + (lane & 7) * 16, r);
        f.b[0][ks][0] = r[0];
        f.b[0][ks][1] = r[1];
        f.b[0][ks + 1][0] = r[2];
        f.b[0][ks + 1][1] = r[3];
      }
    }
  } else {
    static_assert(NT % 2 == 0, "");
#pragma unroll
    for (int nt = 0; nt < NT; nt += 2) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {  // x4 = (chunk 2ks, 2ks+1) x (n-tile nt, nt+1)
        uint32_t r[4];
        const int chunk = 2 * ks + ((lane >> 3) & 1);
        const int n = 8 * nt + (lane & 7) + ((lane >> 4) << 3);
        ldsm4(wbase + off + chunk * npad * 16 + n * 16, r);
        f.b[nt][ks][0] = r[0];
        f.b[nt][ks][1] = r[1];
        f.b[nt + 1][ks][0] = r[2];
        f.b[nt + 1][ks][1] = r[3];
      }
    }
  }
}

// accumulator init from an fp32 bias row [N] (cols 2t, 2t+1 of each n-tile)
template <int NT>
__device__ __forceinline__ void bias_init(uint32_t wbase, uint32_t off, int lane, float (&d)[NT][4]) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const float2 b = lds64f(wbase + off + (8 * nt + 2 * (lane & 3)) * 4);
    d[nt][0] = b.x;
    d[nt][1] = b.y;
    d[nt][2] = b.x;
    d[nt][3] = b.y;
  }
}

// hidden activation -> next layer's A fragments (hi, lo): n-tiles 2j, 2j+1 form k-step j
template <int NT>
__device__ __forceinline__ void split_to_a(const float (&d)[NT][4], uint32_t (&hi)[NT / 2][4],
                                           uint32_t (&lo)[NT / 2][4]) {
#pragma unroll
  for (int j = 0; j < NT / 2; ++j) {
    split_scaled(d[2 * j][0], d[2 * j][1], hi[j][0], lo[j][0]);
    split_scaled(d[2 * j][2], d[2 * j][3], hi[j][1], lo[j][1]);
    split_scaled(d[2 * j + 1][0], d[2 * j + 1][1], hi[j][2], lo[j][2]);
    split_scaled(d[2 * j + 1][2], d[2 * j + 1][3], hi[j][3], lo[j][3]);
  }
}

// one hidden-input layer: D = bias + W (hi + lo)
template <int NTO, int KS>
__device__ __forceinline__ void layer_hl(const uint32_t (&hi)[KS][4], const uint32_t (&lo)[KS][4],
                                         const BFrag<NTO, KS>& B, float (&d)[NTO][4]) {
#pragma unroll
  for (int nt = 0; nt < NTO; ++nt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      mma16(d[nt], hi[ks], B.b[nt][ks][0], B.b[nt][ks][1]);
      mma16(d[nt], lo[ks], B.b[nt][ks][0], B.b[nt][ks][1]);
    }
}

// D fragment (rows 16mt + g / +8, n-tiles) -> stage rows (fp32, 16 per row)
template <int NT>
__device__ __forceinline__ void d_to_stage(uint32_t sb, int mt, int lane, const float (&d)[NT][4],
                                           int max_t = 4) {
  const int g = lane >> 2, t = lane & 3;
  if (t >= max_t) return;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int chunk = 2 * nt + (t >> 1);
    const uint32_t o = 8 * (t & 1);
    sts64f(stg(sb, 16 * mt + g, chunk) + o, d[nt][0], d[nt][1]);
    sts64f(stg(sb, 16 * mt + g + 8, chunk) + o, d[nt][2], d[nt][3]);
  }
}

struct TexPrefetch {
  uint4 tex[4];
  float fx, fy;
  int level;
};

template <int MODE>
__device__ __forceinline__ void prefetch_row(const MatParams& mp, const QueryArgs& a,
                                             const WIn<MODE>& ib, int lane, float lod0,
                                             TexPrefetch& p) {
  const float u = ib.uv[2 * lane], v = ib.uv[2 * lane + 1];
  const float lod = a.lod_stride ? ib.lod[lane] : lod0;
  p.level = choose_level(mp, lod, ib.urr[lane]);
  const Taps t = make_taps(mp, p.level, u, v);
  p.fx = t.fx;
  p.fy = t.fy;
#pragma unroll
  for (int k = 0; k < 4; ++k) p.tex[k] = __ldg(mp.latent + tap_index(t, k));
}

__device__ __forceinline__ void blend_pack(const TexPrefetch& p, uint32_t (&zp)[4]) {
  float2 z[4];
  blend4x2(z, p.tex, p.fx, p.fy);
#pragma unroll
  for (int c = 0; c < 4; ++c) zp[c] = pack2(z[c].x, z[c].y);
}

__device__ __forceinline__ void cp4(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp8(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

// This lane's row of warp tile `wt` into `ib` with cp.async (LDGSTS: no
// registers held, no cross-lane hand-off: every lane reads back only its own
// row); rows past the end get benign defaults.  One commit group per tile.
template <int MODE>
__device__ __forceinline__ void stage_row(const QueryArgs& a, int64_t wt, WIn<MODE>& ib, int lane) {
  const int64_t q = wt * kWT + lane;
  if (q < a.n) {
    cp8(tc::smem_u32(&ib.uv[2 * lane]), a.uv + 2 * q);
    if (a.lod_stride) cp4(tc::smem_u32(&ib.lod[lane]), a.lod + q);
    cp4(tc::smem_u32(&ib.urr[lane]), a.u_rr + q);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cp4(tc::smem_u32(&ib.wi[3 * lane + k]), a.wi + 3 * q + k);
      if constexpr (WNeed<MODE>::wo) cp4(tc::smem_u32(&ib.wo[3 * lane + k]), a.wo + 3 * q + k);
      if constexpr (WNeed<MODE>::u3) cp4(tc::smem_u32(&ib.u3[3 * lane + k]), a.u3 + 3 * q + k);
    }
  } else {
    ib.uv[2 * lane] = ib.uv[2 * lane + 1] = 0.f;
    ib.lod[lane] = ib.urr[lane] = 0.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      ib.wi[3 * lane + k] = k == 2 ? 1.f : 0.f;
      if constexpr (WNeed<MODE>::wo) ib.wo[3 * lane + k] = k == 2 ? 1.f : 0.f;
      if constexpr (WNeed<MODE>::u3) ib.u3[3 * lane + k] = 0.f;
    }
  }
  tc::cp_async_commit();
}

template <int MODE, int BW, int BNH, int SW, int SNH, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
warp_kernel(const __grid_constant__ MatParams mp, const __grid_constant__ QueryArgs a, float inv_brdf,
            float inv_samp) {
  constexpr bool kBrdf = WNeed<MODE>::brdf, kSamp = WNeed<MODE>::samp;
  constexpr int BT = BW / 8;   // BRDF hidden n-tiles
  constexpr int BK = BW / 16;  // BRDF hidden k-steps
  constexpr int ST = SW / 8, SK = SW / 16;
  static_assert(BW % 16 == 0 && SW % 16 == 0, "");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t w_bar;

  const int lane = threadIdx.x & 31;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
  const uint32_t wbytes = (mp.wk_bytes + 127u) & ~127u;
  WIn<MODE>* ibuf = reinterpret_cast<WIn<MODE>*>(smem + wbytes) + warp * 3;
  const uint32_t sbase = tc::smem_u32(smem + wbytes + NW * 3 * sizeof(WIn<MODE>)) + warp * 2048;
  const uint32_t wbase = tc::smem_u32(smem);

  if (threadIdx.x == 0) {
    tc::mbar_init(&w_bar, 1);
    tc::fence_mbar_init();
    tc::mbar_arrive_expect_tx(&w_bar, mp.wk_bytes);
    for (uint32_t o = 0; o < mp.wk_bytes; o += 32768u) {
      const uint32_t nb = mp.wk_bytes - o < 32768u ? mp.wk_bytes - o : 32768u;
      tc::tma_load_1d(tc::smem_u32(smem + o), reinterpret_cast<const uint8_t*>(mp.wk_blob) + o, nb, &w_bar);
    }
  }
  tc::fence_mbar_init();
  __syncthreads();

  const float lod0 = a.lod_stride ? 0.f : __ldg(a.lod);
  const int64_t nwt = (a.n + kWT - 1) / kWT;
  const int64_t wstride = (int64_t)gridDim.x * NW;
  int64_t wt = (int64_t)blockIdx.x * NW + warp;
  const bool want_level = a.level != nullptr;
  const bool want_albedo = mp.albedo && a.albedo;
  const int g = lane >> 2, t4 = lane & 3;

  // prologue: stage tiles 0 and 1 of this warp, fetch + blend tile 0
  uint32_t zp[4];
  int level = 0;
  if (wt < nwt) {
    stage_row<MODE>(a, wt, ibuf[0], lane);
    stage_row<MODE>(a, wt + wstride, ibuf[1], lane);  // (an empty group past the end)
    tc::cp_async_wait<1>();
    TexPrefetch p0;
    prefetch_row<MODE>(mp, a, ibuf[0], lane, lod0, p0);
    blend_pack(p0, zp);
    level = p0.level;
  }
  tc::mbar_wait(&w_bar, 0);

  for (int it = 0; wt < nwt; ++it, wt += wstride) {
    const int b0 = it % 3, b1 = (it + 1) % 3, b2 = (it + 2) % 3;
    const int64_t wt1 = wt + wstride, wt2 = wt + 2 * wstride;
    // (a) tile it+2's inputs into the buffer tile it-1 used (one group per tile)
    if (wt2 < nwt) stage_row<MODE>(a, wt2, ibuf[b2], lane);
    else tc::cp_async_commit();
    // (b) this tile's directions
    const WIn<MODE>& ib = ibuf[b0];
    const V3 wi = v3(ib.wi[3 * lane], ib.wi[3 * lane + 1], ib.wi[3 * lane + 2]);
    V3 wo = v3(0.f, 0.f, 1.f), u3 = v3(0.f, 0.f, 0.f);
    if constexpr (WNeed<MODE>::wo) wo = v3(ib.wo[3 * lane], ib.wo[3 * lane + 1], ib.wo[3 * lane + 2]);
    if constexpr (WNeed<MODE>::u3) u3 = v3(ib.u3[3 * lane], ib.u3[3 * lane + 1], ib.u3[3 * lane + 2]);
    const int64_t q = wt * kWT + lane;
    const bool valid = q < a.n;
    if (want_level) {
      if (valid) a.level[q] = level;
    }
    // (c) next tile's texels: loads now, blended at the end of the iteration
    TexPrefetch nx;
    if (wt1 < nwt) {
      tc::cp_async_wait<1>();  // tile it+1's group (it+2's may still be in flight)
      prefetch_row<MODE>(mp, a, ibuf[b1], lane, lod0, nx);
    }

    // (d) input chunk 0 = [z, wi, 1] -> A0 fragments of both 16-row tiles
    sts128(stg(sbase, lane, 0), zp[0], zp[1], zp[2], zp[3]);
    sts128(stg(sbase, lane, 1), pack2(wi.x, wi.y), pack2(wi.z, 1.f), 0u, 0u);
    __syncwarp();
    uint32_t A0[2][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
      ldsm4(stg(sbase, 16 * mt + (lane & 7) + ((lane >> 3) & 1) * 8, lane >> 4), A0[mt]);
    __syncwarp();

    if constexpr (kBrdf) {
      // (e) frame layer (N = 16) -> rows -> frames, T.wi, T.wo
      {
        BFrag<2, 1> Bf;
        load_b<2, 1>(wbase, mp.wk_fr, lane, Bf);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          float df[2][4] = {};
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) mma16(df[nt], A0[mt], Bf.b[nt][0][0], Bf.b[nt][0][1]);
          d_to_stage<2>(sbase, mt, lane, df);
        }
      }
      __syncwarp();
      float raw[12];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float4 v = lds128f(stg(sbase, lane, c));
        raw[4 * c] = v.x; raw[4 * c + 1] = v.y; raw[4 * c + 2] = v.z; raw[4 * c + 3] = v.w;
      }
      float ti[6], to[6];
      frames2_transform(raw, wi, wo, ti, to);
      __syncwarp();
      // (f) input chunk 1 = [T.wi, T.wo, 1 @ 12] -> A1
      sts128(stg(sbase, lane, 2), pack2(ti[0], ti[1]), pack2(ti[2], ti[3]), pack2(ti[4], ti[5]),
             pack2(to[0], to[1]));
      sts128(stg(sbase, lane, 3), pack2(to[2], to[3]), pack2(to[4], to[5]), 0x00003C00u, 0u);
      __syncwarp();
      uint32_t A1[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
        ldsm4(stg(sbase, 16 * mt + (lane & 7) + ((lane >> 3) & 1) * 8, 2 + (lane >> 4)), A1[mt]);
      __syncwarp();
      // (g) BRDF layers, tile by tile; output D -> stage rows (cols 0-3 / 4-7)
      {
        uint32_t Bz[BT];  // layer 1 on z (K = 8): b0 of each n-tile (rows n = 8 nt + lane)
        if constexpr (BT == 2) {
          ldsm2(wbase + mp.wk_b1z + (lane & 15) * 16, Bz[0], Bz[1]);
        } else {
#pragma unroll
          for (int nt = 0; nt < BT; nt += 4) {
            uint32_t r[4];
            ldsm4(wbase + mp.wk_b1z + (8 * nt + lane) * 16, r);
            Bz[nt] = r[0];
            Bz[nt + 1] = r[1];
            Bz[nt + 2] = r[2];
            Bz[nt + 3] = r[3];
          }
        }
        BFrag<BT, 1> Bt;
        load_b<BT, 1>(wbase, mp.wk_b1t, lane, Bt);
        BFrag<BT, BK> Bh[BNH - 1];
#pragma unroll
        for (int l = 0; l < BNH - 1; ++l) load_b<BT, BK>(wbase, mp.wk_bh[l], lane, Bh[l]);
        BFrag<1, BK> Bo;
        load_b<1, BK>(wbase, mp.wk_bo, lane, Bo);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          float d[BT][4];
#pragma unroll
          for (int nt = 0; nt < BT; ++nt) {
            d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
            mma8(d[nt], A0[mt][0], A0[mt][1], Bz[nt]);
            mma16(d[nt], A1[mt], Bt.b[nt][0][0], Bt.b[nt][0][1]);
          }
#pragma unroll
          for (int l = 0; l < BNH - 1; ++l) {
            uint32_t hi[BK][4], lo[BK][4];
            split_to_a<BT>(d, hi, lo);
            bias_init<BT>(wbase, mp.wk_bias_bh[l], lane, d);
            layer_hl<BT, BK>(hi, lo, Bh[l], d);
          }
          uint32_t hi[BK][4], lo[BK][4];
          split_to_a<BT>(d, hi, lo);
          float o[1][4];
          bias_init<1>(wbase, mp.wk_bias_bo, lane, o);
          layer_hl<1, BK>(hi, lo, Bo, o);
          d_to_stage<1>(sbase, mt, lane, o, 3);
        }
      }
      __syncwarp();
      const float4 y = lds128f(stg(sbase, lane, 0));
      float4 y2 = make_float4(0.f, 0.f, 0.f, 0.f);
      if (want_albedo) y2 = lds128f(stg(sbase, lane, 1));
      if (valid) {
        const bool up = (wi.z > 0.f) && (wo.z > 0.f);
        const V3 f = up ? v3(brdf_output(y.x * inv_brdf), brdf_output(y.y * inv_brdf),
                             brdf_output(y.z * inv_brdf))
                        : v3(0.f, 0.f, 0.f);
        stg3(a.rgb, q, f);
        if (want_albedo) {
          const V3 al = up ? v3(fmaxf(y.w * inv_brdf, 0.f), fmaxf(y2.x * inv_brdf, 0.f),
                                fmaxf(y2.y * inv_brdf, 0.f))
                           : v3(0.f, 0.f, 0.f);
          stg3(a.albedo, q, al);
        }
      }
      __syncwarp();
    }

    if constexpr (kSamp) {
      // (h) sampler decoder on input chunk 0, tile by tile; raw outputs -> stage rows
      {
        BFrag<ST, 1> B1;
        load_b<ST, 1>(wbase, mp.wk_s1, lane, B1);
        BFrag<ST, SK> Bh[SNH - 1];
#pragma unroll
        for (int l = 0; l < SNH - 1; ++l) load_b<ST, SK>(wbase, mp.wk_sh[l], lane, Bh[l]);
        BFrag<2, SK> Bo;
        load_b<2, SK>(wbase, mp.wk_so, lane, Bo);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          float d[ST][4];
#pragma unroll
          for (int nt = 0; nt < ST; ++nt) {
            d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
            mma16(d[nt], A0[mt], B1.b[nt][0][0], B1.b[nt][0][1]);
          }
#pragma unroll
          for (int l = 0; l < SNH - 1; ++l) {
            uint32_t hi[SK][4], lo[SK][4];
            split_to_a<ST>(d, hi, lo);
            bias_init<ST>(wbase, mp.wk_bias_sh[l], lane, d);
            layer_hl<ST, SK>(hi, lo, Bh[l], d);
          }
          uint32_t hi[SK][4], lo[SK][4];
          split_to_a<ST>(d, hi, lo);
          float o[2][4];
          bias_init<2>(wbase, mp.wk_bias_so, lane, o);
          layer_hl<2, SK>(hi, lo, Bo, o);
          d_to_stage<2>(sbase, mt, lane, o);
        }
      }
      __syncwarp();
      float raw[12];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const float4 v = lds128f(stg(sbase, lane, c));
        raw[4 * c] = v.x; raw[4 * c + 1] = v.y; raw[4 * c + 2] = v.z; raw[4 * c + 3] = v.w;
      }
      const Proxy p = proxy_from_raw(raw, mp.isotropic != 0, inv_samp);
      if (valid) {
        if (a.params9) store_proxy(a.params9, q, p);
        const V3 w = proxy_sample(p, wi, u3.x, u3.y, u3.z);
        stg3(a.ws, q, w);
        a.pdf[q] = proxy_pdf(p, wi, w);
      }
      __syncwarp();
    }
    // (i) next tile's latent code
    if (wt1 < nwt) {
      blend_pack(nx, zp);
      level = nx.level;
    }
  }
}

int g_sms_w = 0;

template <int MODE, int BW, int BNH, int SW, int SNH, int NW>
cudaError_t launch_warp_t(const MatParams& mp, const QueryArgs& a, float inv_brdf, float inv_samp,
                          cudaStream_t s) {
  if (!g_sms_w) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms_w, cudaDevAttrMultiProcessorCount, dev);
  }
  auto kern = warp_kernel<MODE, BW, BNH, SW, SNH, NW>;
  const int smem = (int)(((mp.wk_bytes + 127u) & ~127u) + NW * (3 * sizeof(WIn<MODE>) + 2048));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t nwt = (a.n + kWT - 1) / kWT;
  int64_t grid = g_sms_w;
  if (grid > (nwt + NW - 1) / NW) grid = (nwt + NW - 1) / NW;
  if (grid < 1) grid = 1;
  kern<<<(int)grid, NW * 32, smem, s>>>(mp, a, inv_brdf, inv_samp);
  ++g_launches;
  return cudaGetLastError();
}

template <int BW, int BNH, int SW, int SNH>
cudaError_t launch_warp_arch(int mode, const MatParams& mp, const QueryArgs& a, cudaStream_t s) {
  const float ib = (float)(1.0 / std::pow(kLeakyScale, BNH));
  const float is = (float)(1.0 / std::pow(kLeakyScale, SNH));
  switch (mode) {
    case kModeEval: return launch_warp_t<kModeEval, BW, BNH, SW, SNH, NMQ_WARPS>(mp, a, ib, is, s);
    case kModeSamplePdf: return launch_warp_t<kModeSamplePdf, BW, BNH, SW, SNH, NMQ_WARPS>(mp, a, ib, is, s);
    case kModeQuery: return launch_warp_t<kModeQuery, BW, BNH, SW, SNH, NMQ_WARPS>(mp, a, ib, is, s);
    default: return cudaErrorNotSupported;
  }
}

bool aligned16w(const void* p) { return ((uintptr_t)p & 15u) == 0; }

}  // namespace

cudaError_t launch_warp(const MatParams& mp, int mode, const QueryArgs& a, cudaStream_t s) {
  if (mp.fast_arch < 0 || mp.texel_fp32 || a.idx || a.out_idx || a.seg || !mp.wk_blob)
    return cudaErrorNotSupported;
  if (mode != kModeEval && mode != kModeSamplePdf && mode != kModeQuery) return cudaErrorNotSupported;
  if (!aligned16w(a.uv) || !aligned16w(a.u_rr) || !aligned16w(a.wi) ||
      (a.lod_stride && !aligned16w(a.lod)) || (a.wo && !aligned16w(a.wo)) ||
      (a.u3 && !aligned16w(a.u3)))
    return cudaErrorNotSupported;
  switch (mp.fast_arch) {
    case 0: return launch_warp_arch<32, 2, 32, 3>(mode, mp, a, s);
    case 1: return launch_warp_arch<16, 2, 32, 3>(mode, mp, a, s);
    case 2: return launch_warp_arch<64, 3, 32, 3>(mode, mp, a, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace nmq
