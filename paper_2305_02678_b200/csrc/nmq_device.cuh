// nmq_device.cuh — per-query device math of the neural-material query path:
// latent fetch, learned shading frames, proxy parameter maps, sample and pdf.
// One thread owns one query; everything here is scalar SIMT code written
// with MUFU approximations (rsqrt / rcp / ex2 / sin / cos): their ~1e-7
// relative error sits far below the fp16 rounding every value passes through
// before the next network layer, and below the stated tolerances.
// Reference citations: /root/reference/pkg/src/neuralmat/<file>:<line>.
#pragma once
#include <cstdint>
#include <cuda_fp16.h>
#include "nmq_internal.h"

namespace nmq {
namespace dev {

constexpr float kPi = 3.14159265358979323846f;
constexpr float kInvPi = 0.31830988618379067154f;
constexpr float kLog2e = 1.44269504088896340736f;
constexpr float kAlphaFloor = 1e-4f;               // proxy.py:32
constexpr float kRhoClamp = 0.99994999874993749f;  // sqrt(1 - 1e-4), proxy.py:33
constexpr float kLeaky = 0.01f;                    // mlp.py:16

struct V3 {
  float x, y, z;
};
__device__ __forceinline__ V3 v3(float x, float y, float z) { return {x, y, z}; }
__device__ __forceinline__ float dot(V3 a, V3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
__device__ __forceinline__ V3 cross(V3 a, V3 b) {
  return {fmaf(a.y, b.z, -a.z * b.y), fmaf(a.z, b.x, -a.x * b.z), fmaf(a.x, b.y, -a.y * b.x)};
}
__device__ __forceinline__ V3 scale(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }

// approximate helpers (MUFU)
__device__ __forceinline__ float rcp(float x) { return __fdividef(1.f, x); }
__device__ __forceinline__ float fsqrt(float x) {  // sqrt via rsqrt, exact 0 at 0
  return x > 0.f ? x * rsqrtf(x) : 0.f;
}
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ V3 ldg3(const float* p, int64_t i) {
  return {__ldg(p + 3 * i), __ldg(p + 3 * i + 1), __ldg(p + 3 * i + 2)};
}
__device__ __forceinline__ void stg3(float* p, int64_t i, V3 v) {
  p[3 * i] = v.x;
  p[3 * i + 1] = v.y;
  p[3 * i + 2] = v.z;
}

// ---------------------------------------------------------------------------
// Latent fetch.  choose_level (latent.py:76-82) is exact in fp32 for fp32
// inputs (clip/floor/subtract of a float are exact).  Texel coordinates
// follow _taps (latent.py:56-74): for power-of-two level sizes u*w is exact
// in fp32 and the floor/half-texel decision below is exact; otherwise the
// coordinate is computed in float64 like the reference.  Either way the
// level and the four tap indices are bit-identical to the reference.  The
// blend is fp32 FMA over the stored texels (the reference sums in float64
// and rounds to fp32).
struct Taps {
  int64_t base;  // texel index of the level origin
  int32_t x0, x1, y0, y1, w;
  float fx, fy;
};

__device__ __forceinline__ int choose_level(const MatParams& m, float lod, float urr) {
  const float top = (float)(m.n_levels - 1);
  float l = fminf(fmaxf(lod, 0.f), top);
  const float lo = floorf(l);
  int c = (int)lo + ((urr < (l - lo)) ? 1 : 0);
  c = c < 0 ? 0 : c;
  c = c > m.n_levels - 1 ? m.n_levels - 1 : c;
  return c;
}

__device__ __forceinline__ int64_t wrap_index(double f, int32_t n) {
  // Python's non-negative modulo of floor(f) (latent.py:65-68)
  const int64_t i = (int64_t)f;
  int64_t r = i % n;
  return r < 0 ? r + n : r;
}

// exact floor(u*w - 0.5) and its fraction for power-of-two w (u*w is exact)
__device__ __forceinline__ void axis_pow2(float u, int32_t w, int32_t& i0, float& f) {
  const float t = u * (float)w;  // exact: scaling by a power of two
  const float ti = floorf(t);
  const float fr = t - ti;       // exact
  const bool lo = fr < 0.5f;
  i0 = ((int32_t)(int64_t)ti - (lo ? 1 : 0)) & (w - 1);
  f = lo ? fr + 0.5f : fr - 0.5f;
}

__device__ __forceinline__ Taps make_taps(const MatParams& m, int level, float u, float v) {
  const LevelDesc L = m.lv[level];
  Taps t;
  if (m.pow2) {
    axis_pow2(u, L.w, t.x0, t.fx);
    axis_pow2(v, L.h, t.y0, t.fy);
  } else {
    const double x = fma((double)u, (double)L.w, -0.5);
    const double y = fma((double)v, (double)L.h, -0.5);
    const double xf = floor(x), yf = floor(y);
    t.fx = (float)(x - xf);
    t.fy = (float)(y - yf);
    t.x0 = (int32_t)wrap_index(xf, L.w);
    t.y0 = (int32_t)wrap_index(yf, L.h);
  }
  t.x1 = (t.x0 + 1 == L.w) ? 0 : t.x0 + 1;
  t.y1 = (t.y0 + 1 == L.h) ? 0 : t.y0 + 1;
  t.w = L.w;
  t.base = L.off;
  return t;
}

__device__ __forceinline__ int64_t tap_index(const Taps& t, int k) {
  const int32_t x = (k & 1) ? t.x1 : t.x0;
  const int32_t y = (k & 2) ? t.y1 : t.y0;
  return t.base + (int64_t)y * t.w + x;
}

__device__ __forceinline__ void blend_texel(float (&z)[8], uint4 t, float w) {
  const __half2* h = reinterpret_cast<const __half2*>(&t);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = __half22float2(h[k]);
    z[2 * k] = fmaf(f.x, w, z[2 * k]);
    z[2 * k + 1] = fmaf(f.y, w, z[2 * k + 1]);
  }
}

__device__ __forceinline__ void blend4(float (&z)[8], const uint4 (&tex)[4], float fx, float fy) {
  const float gx = 1.f - fx, gy = 1.f - fy;
#pragma unroll
  for (int k = 0; k < 8; ++k) z[k] = 0.f;
  blend_texel(z, tex[0], gx * gy);
  blend_texel(z, tex[1], fx * gy);
  blend_texel(z, tex[2], gx * fy);
  blend_texel(z, tex[3], fx * fy);
}

// ---- packed fp32x2 (FFMA2 / FMUL2, sm_100) -----------------------------------
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2s(float2 a, float s, float2 c) {
  return __ffma2_rn(a, make_float2(s, s), c);
}
__device__ __forceinline__ float2 mul2s(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }

// Bilinear blend with z as four channel pairs: 16 FFMA2 instead of 32 FFMA.
__device__ __forceinline__ void blend4x2(float2 (&z)[4], const uint4 (&tex)[4], float fx, float fy) {
  const float gx = 1.f - fx, gy = 1.f - fy;
  const float w[4] = {gx * gy, fx * gy, gx * fy, fx * fy};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const __half2* h = reinterpret_cast<const __half2*>(&tex[k]);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float2 f = __half22float2(h[c]);
      z[c] = k == 0 ? mul2s(f, w[0]) : fma2s(f, w[k], z[c]);
    }
  }
}

// Two 3-vectors held component-wise as pairs (lane .x = first, .y = second).
struct V3x2 {
  float2 x, y, z;
};
__device__ __forceinline__ float2 dot2(const V3x2& a, const V3x2& b) {
  return fma2(a.x, b.x, fma2(a.y, b.y, mul2(a.z, b.z)));
}
__device__ __forceinline__ float2 dot2s(const V3x2& a, V3 w) {  // (a1.w, a2.w)
  return fma2s(a.x, w.x, fma2s(a.y, w.y, mul2s(a.z, w.z)));
}
__device__ __forceinline__ V3x2 cross2(const V3x2& a, const V3x2& b) {
  return {fma2(a.y, b.z, mul2(neg2(a.z), b.y)), fma2(a.z, b.x, mul2(neg2(a.x), b.z)),
          fma2(a.x, b.y, mul2(neg2(a.y), b.x))};
}
__device__ __forceinline__ V3x2 scale2(const V3x2& a, float2 s) {
  return {mul2(a.x, s), mul2(a.y, s), mul2(a.z, s)};
}

__device__ __forceinline__ void blend_texel32(float (&z)[8], const float4* p, float w) {
  const float4 a = __ldg(p), b = __ldg(p + 1);
  z[0] = fmaf(a.x, w, z[0]); z[1] = fmaf(a.y, w, z[1]);
  z[2] = fmaf(a.z, w, z[2]); z[3] = fmaf(a.w, w, z[3]);
  z[4] = fmaf(b.x, w, z[4]); z[5] = fmaf(b.y, w, z[5]);
  z[6] = fmaf(b.z, w, z[6]); z[7] = fmaf(b.w, w, z[7]);
}

// Bilinear fetch of 8 channels straight from global memory (4 x LDG.128).
__device__ __forceinline__ void fetch_taps(const MatParams& m, const Taps& t, float (&z)[8]) {
  if (m.texel_fp32) {  // generic fp32 pyramid (LatentPyramid master copy)
    const float4* lat = reinterpret_cast<const float4*>(m.latent);
    const float gx = 1.f - t.fx, gy = 1.f - t.fy;
#pragma unroll
    for (int k = 0; k < 8; ++k) z[k] = 0.f;
    blend_texel32(z, lat + 2 * tap_index(t, 0), gx * gy);
    blend_texel32(z, lat + 2 * tap_index(t, 1), t.fx * gy);
    blend_texel32(z, lat + 2 * tap_index(t, 2), gx * t.fy);
    blend_texel32(z, lat + 2 * tap_index(t, 3), t.fx * t.fy);
    return;
  }
  uint4 tex[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) tex[k] = __ldg(m.latent + tap_index(t, k));
  blend4(z, tex, t.fx, t.fy);
}

// ---------------------------------------------------------------------------
// Learned shading frame (neural.py:207-233 + geom.py:82-89 fallback).
struct Frame {
  V3 t, b, n;
};

__device__ __forceinline__ V3 fallback_tangent(V3 n) {
  // n x e_k, k = argmin |n_k| (first index on ties), normalized
  const float ax = fabsf(n.x), ay = fabsf(n.y), az = fabsf(n.z);
  V3 e;
  if (ax <= ay && ax <= az) e = v3(1.f, 0.f, 0.f);
  else if (ay <= az) e = v3(0.f, 1.f, 0.f);
  else e = v3(0.f, 0.f, 1.f);
  V3 c = cross(n, e);
  return scale(c, rsqrtf(dot(c, c)));
}

__device__ __forceinline__ Frame frame_from_raw(const float* r) {
  const V3 rn = v3(r[0], r[1], r[2]);
  V3 rt = v3(r[3], r[4], r[5]);
  // n = rn / max(|rn|, 1e-12)
  const V3 n = scale(rn, rsqrtf(fmaxf(dot(rn, rn), 1e-24f)));
  V3 c = cross(n, rt);
  float c2 = dot(c, c);
  if (c2 < 1e-16f) {  // |c| < 1e-8: degenerate tangent
    rt = fallback_tangent(n);
    c = cross(n, rt);
    c2 = dot(c, c);
  }
  Frame f;
  f.b = scale(c, rsqrtf(fmaxf(c2, 1e-24f)));
  f.n = n;
  f.t = cross(f.b, n);
  return f;
}

// Both learned frames at once (neural.py:207-233) with packed fp32x2 math,
// and the direction transforms T.wi, T.wo (neural.py:185-196):
// ti = [t1.wi, b1.wi, n1.wi, t2.wi, b2.wi, n2.wi], same for to.  Returns
// each frame's conditioning kappa = 1 + |rt|_1 / |n x rt| (the fp32 error
// of b and t grows as 1/|n x rt|), +inf near the reference's
// degenerate-tangent branch or a vanishing normal (resolved exactly).
__device__ __forceinline__ float2 frames2_transform(const float* r, V3 wi, V3 wo, float (&ti)[6],
                                                    float (&to)[6]) {
  const V3x2 rn = {f2(r[0], r[6]), f2(r[1], r[7]), f2(r[2], r[8])};
  V3x2 rt = {f2(r[3], r[9]), f2(r[4], r[10]), f2(r[5], r[11])};
  const float2 l2 = dot2(rn, rn);
  const V3x2 n = scale2(rn, f2(rsqrtf(fmaxf(l2.x, 1e-24f)), rsqrtf(fmaxf(l2.y, 1e-24f))));
  const float2 rt1 = __fadd2_rn(__fadd2_rn(f2(fabsf(rt.x.x), fabsf(rt.x.y)), f2(fabsf(rt.y.x), fabsf(rt.y.y))),
                                f2(fabsf(rt.z.x), fabsf(rt.z.y)));
  V3x2 c = cross2(n, rt);
  float2 c2 = dot2(c, c);
  const bool ill1 = c2.x < 1e-10f || l2.x < 1e-20f, ill2 = c2.y < 1e-10f || l2.y < 1e-20f;
  if (c2.x < 1e-16f || c2.y < 1e-16f) {  // |c| < 1e-8: degenerate tangent(s)
    if (c2.x < 1e-16f) {
      const V3 f = fallback_tangent(v3(n.x.x, n.y.x, n.z.x));
      rt.x.x = f.x; rt.y.x = f.y; rt.z.x = f.z;
    }
    if (c2.y < 1e-16f) {
      const V3 f = fallback_tangent(v3(n.x.y, n.y.y, n.z.y));
      rt.x.y = f.x; rt.y.y = f.y; rt.z.y = f.z;
    }
    c = cross2(n, rt);
    c2 = dot2(c, c);
  }
  const float2 ic = f2(rsqrtf(fmaxf(c2.x, 1e-24f)), rsqrtf(fmaxf(c2.y, 1e-24f)));
  const V3x2 b = scale2(c, ic);
  const V3x2 t = cross2(b, n);
  const float2 twi = dot2s(t, wi), bwi = dot2s(b, wi), nwi = dot2s(n, wi);
  const float2 two = dot2s(t, wo), bwo = dot2s(b, wo), nwo = dot2s(n, wo);
  ti[0] = twi.x; ti[1] = bwi.x; ti[2] = nwi.x; ti[3] = twi.y; ti[4] = bwi.y; ti[5] = nwi.y;
  to[0] = two.x; to[1] = bwo.x; to[2] = nwo.x; to[3] = two.y; to[4] = bwo.y; to[5] = nwo.y;
  const float2 kap = __ffma2_rn(rt1, ic, f2(1.f, 1.f));
  return f2(ill1 ? __int_as_float(0x7f800000) : kap.x, ill2 ? __int_as_float(0x7f800000) : kap.y);
}

// ---------------------------------------------------------------------------
// BRDF output map (neural.py:37-39): max(expm1(min(y, 60)), 0)
__device__ __forceinline__ float brdf_output(float y) {
  return y > 0.f ? ex2(fminf(y, 60.f) * kLog2e) - 1.f : 0.f;
}

// ---------------------------------------------------------------------------
// Proxy parameter maps (neural.py:46-71, 317-331) and floors (proxy.py:42-50)
__device__ __forceinline__ float quad_tanh(float x) {
  const float ax = fabsf(x);
  if (ax > 1e18f) return copysignf(1.f, x);
  const float r = __fdividef(x * fmaf(0.5f, ax, 1.f), fmaf(0.5f * x, x, 1.f + ax));
  return fminf(fmaxf(r, -1.f), 1.f);
}
__device__ __forceinline__ float quad_sinh(float x) { return x * fmaf(x * x, 1.f / 6.f, 1.f); }

struct Proxy {
  float wd, ws, mdx, mdy, ax, ay, rho, msx, msy;
};

// raw outputs may arrive scaled by `s` (the MLP engine's leaky rescaling)
__device__ __forceinline__ Proxy proxy_from_raw(const float* raw, bool isotropic, float s = 1.f) {
  Proxy p;
  if (isotropic) {
    p.wd = 0.5f * (quad_tanh(raw[0] * s) + 1.f);
    p.ws = 1.f - p.wd;
    const float a = 0.5f * (quad_tanh(raw[1] * s) + 1.f);
    p.ax = p.ay = a;
    p.mdx = p.mdy = p.rho = p.msx = p.msy = 0.f;
  } else {
    const float a = raw[0] * s, b = raw[3] * s;
    const float m = fmaxf(a, b);
    const float ea = ex2((a - m) * kLog2e), eb = ex2((b - m) * kLog2e);
    const float inv = rcp(ea + eb);
    p.wd = ea * inv;
    p.ws = eb * inv;
    p.mdx = quad_sinh(raw[1] * s);
    p.mdy = quad_sinh(raw[2] * s);
    p.ax = 0.5f * (quad_tanh(raw[4] * s) + 1.f);
    p.ay = 0.5f * (quad_tanh(raw[5] * s) + 1.f);
    p.rho = quad_tanh(raw[6] * s);
    p.msx = quad_sinh(raw[7] * s);
    p.msy = quad_sinh(raw[8] * s);
  }
  p.ax = fmaxf(p.ax, kAlphaFloor);
  p.ay = fmaxf(p.ay, kAlphaFloor);
  p.rho = fminf(fmaxf(p.rho, -kRhoClamp), kRhoClamp);
  return p;
}

__device__ __forceinline__ Proxy load_proxy(const float* p9, int64_t i) {
  const float* q = p9 + 9 * i;
  Proxy p;
  p.wd = __ldg(q + 0); p.ws = __ldg(q + 1);
  p.mdx = __ldg(q + 2); p.mdy = __ldg(q + 3);
  p.ax = fmaxf(__ldg(q + 4), kAlphaFloor); p.ay = fmaxf(__ldg(q + 5), kAlphaFloor);
  p.rho = fminf(fmaxf(__ldg(q + 6), -kRhoClamp), kRhoClamp);
  p.msx = __ldg(q + 7); p.msy = __ldg(q + 8);
  return p;
}
__device__ __forceinline__ void store_proxy(float* p9, int64_t i, const Proxy& p) {
  float* q = p9 + 9 * i;
  q[0] = p.wd; q[1] = p.ws; q[2] = p.mdx; q[3] = p.mdy; q[4] = p.ax;
  q[5] = p.ay; q[6] = p.rho; q[7] = p.msx; q[8] = p.msy;
}

__device__ __forceinline__ float proxy_s(const Proxy& p) {
  // sqrt(1 - rho^2) written as sqrt((1-rho)(1+rho)) for accuracy near |rho|=1
  return fsqrt((1.f - p.rho) * (1.f + p.rho));
}

__device__ __forceinline__ V3 diffuse_axis(const Proxy& p) {
  const V3 v = v3(-p.mdx, -p.mdy, 1.f);
  return scale(v, rsqrtf(dot(v, v)));
}

// proxy.py:114-135
__device__ __forceinline__ float proxy_pdf(const Proxy& p, V3 wi, V3 wo) {
  const V3 nd = diffuse_axis(p);
  const float pd = fmaxf(dot(wo, nd), 0.f) * kInvPi;
  float ps = 0.f;
  V3 h = add(wi, wo);
  const float hl2 = dot(h, h);
  if (hl2 > 1e-18f) {  // |wi + wo| > 1e-9
    h = scale(h, rsqrtf(hl2));
    if (h.z < 0.f) h = scale(h, -1.f);
    if (h.z > 0.f) {
      const float s = proxy_s(p);
      const float q0 = fmaf(p.msx, h.z, h.x) * rcp(p.ax);
      const float q1 = fmaf(fmaf(p.msy, h.z, h.y), rcp(p.ay), -p.rho * q0) * rcp(s);
      const float q2 = fmaf(q0, q0, fmaf(q1, q1, h.z * h.z));
      const float coh = fmaxf(fabsf(dot(wo, h)), 1e-12f);
      const float det = p.ax * p.ay * s;
      ps = fmaxf(__fdividef(h.z, det * (4.f * kPi) * q2 * q2 * coh), 0.f);
    }
  }
  return fmaf(p.wd, pd, p.ws * ps);
}

// proxy.py:138-180.  sqrt(1-cos^2) rewritten as sqrt(tan2)*cos and
// sqrt(1-z^2) as 2 sqrt(u(1-u)) (same values, no cancellation).
__device__ __forceinline__ V3 proxy_sample(const Proxy& p, V3 wi, float u0, float u1, float u2) {
  float sp, cp;
  __sincosf(2.f * kPi * u2, &sp, &cp);
  if (u0 < p.wd) {
    // diffuse: normalize(n_d + uniform_sphere(u1,u2)), |.| floor 1e-9
    const float z = fmaf(-2.f, u1, 1.f);
    const float r = 2.f * fsqrt(u1 * (1.f - u1));
    const V3 g = add(diffuse_axis(p), v3(r * cp, r * sp, z));
    return scale(g, rsqrtf(fmaxf(dot(g, g), 1e-18f)));
  }
  const float tan2 = u1 * rcp(fmaxf(1.f - u1, 1e-12f));
  const float ct = rsqrtf(1.f + tan2);
  const float st = fsqrt(tan2) * ct;
  const V3 m = v3(st * cp, st * sp, ct);
  const float s = proxy_s(p);
  // g = M m, M = [[ax, 0, -msx], [ay rho, ay s, -msy], [0, 0, 1]]
  const V3 g = v3(fmaf(p.ax, m.x, -p.msx * m.z),
                  fmaf(p.ay * p.rho, m.x, fmaf(p.ay * s, m.y, -p.msy * m.z)), m.z);
  const V3 h = scale(g, rsqrtf(fmaxf(dot(g, g), 1e-24f)));
  const float d = 2.f * dot(wi, h);
  return v3(fmaf(d, h.x, -wi.x), fmaf(d, h.y, -wi.y), fmaf(d, h.z, -wi.z));
}

// ---------------------------------------------------------------------------
// Exact-rounding helpers.  The reference's fp16 path rounds
// every decoder input to fp16 once (mlp.py:205) after computing it in
// float64 and narrowing to fp32 (latent.py:93-97, neural.py:282-287):
// z = fp32(sum_k t_k w_k), T.w = fp32(f64 frames . w).  To reproduce those
// fp16 values bit for bit the latent blend runs in float64 and the frame
// transform is resolved in float64 wherever the fast fp32 value lies within
// its error bound of an fp16 rounding midpoint.

// fractional texel coordinate of one axis, float64 (latent.py:59-64): u*w is
// exact in float64 for fp32 u, so fma(u, w, -0.5) == fl(u*w - 0.5)
__device__ __forceinline__ double frac64(float u, int32_t w) {
  const double x = fma((double)u, (double)w, -0.5);
  return x - floor(x);
}

// bilinear weights [(1-fx)(1-fy), fx(1-fy), (1-fx)fy, fx fy] (latent.py:69-71)
__device__ __forceinline__ void weights64(double fx, double fy, double (&w)[4]) {
  const double gx = __dsub_rn(1.0, fx), gy = __dsub_rn(1.0, fy);
  w[0] = __dmul_rn(gx, gy);
  w[1] = __dmul_rn(fx, gy);
  w[2] = __dmul_rn(gx, fy);
  w[3] = __dmul_rn(fx, fy);
}

__device__ __forceinline__ double h2d_lo(uint32_t v) {
  double d;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f64.f16 %0, l;\n\t}" : "=d"(d) : "r"(v));
  return d;
}
__device__ __forceinline__ double h2d_hi(uint32_t v) {
  double d;
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %1;\n\tcvt.f64.f16 %0, h;\n\t}" : "=d"(d) : "r"(v));
  return d;
}

// z = fp32(((t0 w0 + t1 w1) + t2 w2) + t3 w3) with the reference's float64
// rounding of every product and sum (numpy reduces the tap axis left to
// right): bit-identical to latent.py:96.  FMA = true contracts each
// product into its sum (one rounding less; the fp32 result differs only if
// the float64 sum lies within 2^-53 of an fp32 rounding midpoint).
template <bool FMA>
__device__ __forceinline__ void blend64(const uint4 (&tex)[4], const double (&w)[4], float (&z)[8]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = (&tex[k].x)[c];
      const double a = h2d_lo(v), b = h2d_hi(v);
      if (k == 0) {
        s0 = __dmul_rn(a, w[0]);
        s1 = __dmul_rn(b, w[0]);
      } else if (FMA) {
        s0 = fma(a, w[k], s0);
        s1 = fma(b, w[k], s1);
      } else {
        s0 = __dadd_rn(s0, __dmul_rn(a, w[k]));
        s1 = __dadd_rn(s1, __dmul_rn(b, w[k]));
      }
    }
    z[2 * c] = (float)s0;
    z[2 * c + 1] = (float)s1;
  }
}

// fp32 texels (the fp32 master pyramid of the reference's fp32 path)
__device__ __forceinline__ void blend64_f32(const float4* lat, const int64_t (&idx)[4],
                                            const double (&w)[4], float (&z)[8]) {
  double s[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 a = __ldg(lat + 2 * idx[k]), b = __ldg(lat + 2 * idx[k] + 1);
    const float t[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double p = __dmul_rn((double)t[c], w[k]);
      s[c] = k == 0 ? p : __dadd_rn(s[c], p);
    }
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) z[c] = (float)s[c];
}

// Exact fetch (latent.py:84-98): float64 weights and blend, fp32 result.
__device__ __forceinline__ void fetch_exact(const MatParams& m, int level, float u, float v, const Taps& t,
                                            float (&z)[8]) {
  double w[4];
  weights64(frac64(u, m.lv[level].w), frac64(v, m.lv[level].h), w);
  if (m.texel_fp32) {
    const int64_t idx[4] = {tap_index(t, 0), tap_index(t, 1), tap_index(t, 2), tap_index(t, 3)};
    blend64_f32(reinterpret_cast<const float4*>(m.latent), idx, w, z);
    return;
  }
  uint4 tex[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) tex[k] = __ldg(m.latent + tap_index(t, k));
  blend64<false>(tex, w, z);
}

// float64 coordinates (the reference's own dtype: uv, level and u_rr are
// float64 arrays in latent.py / render.py:369) — every step as numpy does it
__device__ __forceinline__ int choose_level(const MatParams& m, double lod, double urr) {
  const double top = (double)(m.n_levels - 1);
  const double l = fmin(fmax(lod, 0.0), top);
  const double lo = floor(l);
  int c = (int)lo + ((urr < __dsub_rn(l, lo)) ? 1 : 0);
  c = c < 0 ? 0 : c;
  c = c > m.n_levels - 1 ? m.n_levels - 1 : c;
  return c;
}
__device__ __forceinline__ double frac64d(double u, int32_t w) {  // latent.py:59-64: fl(fl(u*w) - 0.5)
  const double x = __dsub_rn(__dmul_rn(u, (double)w), 0.5);
  return __dsub_rn(x, floor(x));
}
__device__ __forceinline__ Taps make_taps(const MatParams& m, int level, double u, double v) {
  const LevelDesc L = m.lv[level];
  Taps t;
  const double x = __dsub_rn(__dmul_rn(u, (double)L.w), 0.5);
  const double y = __dsub_rn(__dmul_rn(v, (double)L.h), 0.5);
  const double xf = floor(x), yf = floor(y);
  t.fx = (float)(x - xf);
  t.fy = (float)(y - yf);
  t.x0 = (int32_t)wrap_index(xf, L.w);
  t.y0 = (int32_t)wrap_index(yf, L.h);
  t.x1 = (t.x0 + 1 == L.w) ? 0 : t.x0 + 1;
  t.y1 = (t.y0 + 1 == L.h) ? 0 : t.y0 + 1;
  t.w = L.w;
  t.base = L.off;
  return t;
}
__device__ __forceinline__ void fetch_exact(const MatParams& m, int level, double u, double v, const Taps& t,
                                            float (&z)[8]) {
  double w[4];
  weights64(frac64d(u, m.lv[level].w), frac64d(v, m.lv[level].h), w);
  if (m.texel_fp32) {
    const int64_t idx[4] = {tap_index(t, 0), tap_index(t, 1), tap_index(t, 2), tap_index(t, 3)};
    blend64_f32(reinterpret_cast<const float4*>(m.latent), idx, w, z);
    return;
  }
  uint4 tex[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) tex[k] = __ldg(m.latent + tap_index(t, k));
  blend64<false>(tex, w, z);
}

// fp16 rounding of a pair (the decoder input rounding, mlp.py:205)
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float2 unpack_h2(uint32_t v) {
  return __half22float2(*reinterpret_cast<const __half2*>(&v));
}

// Frame layer on the CUDA cores in the reference's arithmetic: numpy's
// fp32 `x @ W.T` (OpenBLAS sgemm: one fused multiply-add per k, k = 0..7,
// in order; pinned by tests/test_oracle_golden.py) then `+ b` (mlp.py:207).
// x = the fp16 latent code (4 packed pairs).
__device__ __forceinline__ void frame_raw_seq(const MatParams& m, const uint32_t (&zh)[4], float (&raw)[12]) {
  float x[8];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float2 f = unpack_h2(zh[c]);
    x[2 * c] = f.x;
    x[2 * c + 1] = f.y;
  }
  // output j of both frames at once (two independent fp32 FMA chains per FFMA2)
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    float2 acc = __fmul2_rn(make_float2(x[0], x[0]), m.fw2[j][0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) acc = __ffma2_rn(make_float2(x[k], x[k]), m.fw2[j][k], acc);
    acc = __fadd2_rn(acc, m.fw2[j][8]);
    raw[j] = acc.x;
    raw[j + 6] = acc.y;
  }
}

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 d3(V3 v) { return {v.x, v.y, v.z}; }
// numpy's float64 operations, operation for operation (every product and sum
// rounded separately — the _rn intrinsics are never contracted into DFMA):
//   np.sum(a * b, axis=-1) over 3 values: (p0 + p1) + p2
//   np.linalg.norm(v, axis=-1) = sqrt(add.reduce(v * v))
//   np.cross(a, b)[0] = a1*b2 - a2*b1, [1] = a2*b0 - a0*b2, [2] = a0*b1 - a1*b0
//   v / s: IEEE division
__device__ __forceinline__ double np_dot(D3 a, D3 b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ double np_norm(D3 v) { return __dsqrt_rn(np_dot(v, v)); }
__device__ __forceinline__ D3 np_cross(D3 a, D3 b) {
  return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)), __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
          __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ D3 np_div(D3 v, double s) { return {__ddiv_rn(v.x, s), __ddiv_rn(v.y, s), __ddiv_rn(v.z, s)}; }

// One learned frame in float64 and the transform of wi / wo, bit for bit as
// numpy computes them (frames_from_raw, neural.py:207-233; fallback_tangent,
// geom.py:82-89; FrameSet.transform, neural.py:185-196), rounded to fp32 as
// the reference's `inp.astype(np.float32)` does (neural.py:287).
__device__ __forceinline__ void frame_tw64(const float* raw, D3 di, D3 dout, float (&ti)[3], float (&to)[3]) {
  const D3 rn = {raw[0], raw[1], raw[2]};
  D3 rt = {raw[3], raw[4], raw[5]};
  const D3 n = np_div(rn, fmax(np_norm(rn), 1e-12));
  D3 c = np_cross(n, rt);
  double c_len = np_norm(c);
  if (c_len < 1e-8) {  // degenerate: tangent n x e, e the axis of the smallest |n_k| (first on ties)
    const double ax = fabs(n.x), ay = fabs(n.y), az = fabs(n.z);
    const D3 e = (ax <= ay && ax <= az) ? D3{1.0, 0.0, 0.0} : (ay <= az ? D3{0.0, 1.0, 0.0} : D3{0.0, 0.0, 1.0});
    const D3 f = np_cross(n, e);
    rt = np_div(f, np_norm(f));
    c = np_cross(n, rt);
    c_len = np_norm(c);
  }
  const D3 b = np_div(c, fmax(c_len, 1e-12));
  const D3 t = np_cross(b, n);
  ti[0] = (float)np_dot(t, di); ti[1] = (float)np_dot(b, di); ti[2] = (float)np_dot(n, di);
  to[0] = (float)np_dot(t, dout); to[1] = (float)np_dot(b, dout); to[2] = (float)np_dot(n, dout);
}

__device__ __forceinline__ void pack_tw(const MatParams& m, const float (&ti)[6], const float (&to)[6],
                                        uint32_t (&x16)[6]) {
  if (m.n_frames == 2) {
    x16[0] = pack_h2(ti[0], ti[1]); x16[1] = pack_h2(ti[2], ti[3]); x16[2] = pack_h2(ti[4], ti[5]);
    x16[3] = pack_h2(to[0], to[1]); x16[4] = pack_h2(to[2], to[3]); x16[5] = pack_h2(to[4], to[5]);
  } else {  // [T.wi(3), T.wo(3)]
    x16[0] = pack_h2(ti[0], ti[1]); x16[1] = pack_h2(ti[2], to[0]); x16[2] = pack_h2(to[1], to[2]);
    x16[3] = x16[4] = x16[5] = 0u;
  }
}

// The decoder's direction inputs, exactly as the reference rounds them:
// x16 = fp16 pairs of [T.wi (3 per frame), T.wo (3 per frame)] for n_frames
// frames, from the latent code's fp16 pairs.
__device__ __forceinline__ void tw_exact(const MatParams& m, const uint32_t (&zh)[4], D3 wi, D3 wo,
                                         uint32_t (&x16)[6], uint32_t frames = 3u) {
  float raw[12];
  frame_raw_seq(m, zh, raw);
  float ti[6], to[6];
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    if (f < m.n_frames && ((frames >> f) & 1u)) {
      float a[3], b[3];
      frame_tw64(raw + 6 * f, wi, wo, a, b);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        ti[3 * f + k] = a[k];
        to[3 * f + k] = b[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) ti[3 * f + k] = to[3 * f + k] = 0.f;
    }
  }
  pack_tw(m, ti, to, x16);
}
__device__ __forceinline__ void tw_exact(const MatParams& m, const uint32_t (&zh)[4], V3 wi, V3 wo,
                                         uint32_t (&x16)[6], uint32_t frames = 3u) {
  tw_exact(m, zh, d3(wi), d3(wo), x16, frames);
}

// ---- the fast kernel's resolve ------------------------------------------------
// The same frame and transform in float64 by reciprocal square roots and
// FMA-contracted products (the form the fast kernel's epilogue resolve
// uses: numpy's IEEE divisions and square roots cost it 5 % of C2 through
// register pressure in the shared kernel — measured).  Its float64 values
// are within ~20 kappa ulp of numpy's (kappa = 1 + |r_t|_1 / |n x r_t|):
// the fp16 result can differ from numpy's only when a value lies that close
// to an fp32 rounding midpoint which also decides its fp16 rounding (~1e-13
// per value); tests/test_gpu_scale.py checks whole C2 batches row by row.
__device__ __forceinline__ double drsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  return y * fma(-h * y, y, 1.5);
}
__device__ __forceinline__ double fdot(D3 a, D3 b) { return fma(a.z, b.z, fma(a.y, b.y, a.x * b.x)); }
__device__ __forceinline__ D3 fcross(D3 a, D3 b) {
  return {fma(a.y, b.z, -a.z * b.y), fma(a.z, b.x, -a.x * b.z), fma(a.x, b.y, -a.y * b.x)};
}
__device__ __forceinline__ D3 fscale(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ void frame_tw64_rsq(const float* raw, D3 di, D3 dout, float (&ti)[3], float (&to)[3]) {
  const D3 rn = {raw[0], raw[1], raw[2]};
  D3 rt = {raw[3], raw[4], raw[5]};
  const D3 n = fscale(rn, drsqrt(fmax(fdot(rn, rn), 1e-24)));
  D3 c = fcross(n, rt);
  double c2 = fdot(c, c);
  if (c2 < 1e-16) {  // |c| < 1e-8: fallback tangent n x e_argmin|n| (first index on ties)
    const double ax = fabs(n.x), ay = fabs(n.y), az = fabs(n.z);
    const D3 e = (ax <= ay && ax <= az) ? D3{1.0, 0.0, 0.0} : (ay <= az ? D3{0.0, 1.0, 0.0} : D3{0.0, 0.0, 1.0});
    const D3 f = fcross(n, e);
    rt = fscale(f, drsqrt(fdot(f, f)));
    c = fcross(n, rt);
    c2 = fdot(c, c);
  }
  const D3 b = fscale(c, drsqrt(fmax(c2, 1e-24)));
  const D3 t = fcross(b, n);
  ti[0] = (float)fdot(t, di); ti[1] = (float)fdot(b, di); ti[2] = (float)fdot(n, di);
  to[0] = (float)fdot(t, dout); to[1] = (float)fdot(b, dout); to[2] = (float)fdot(n, dout);
}
// frames: THIS row's frames to compute (bit f = frame f).  The float64
// frame runs once per pass for all lanes of the warp, each lane on its own
// next frame — a warp whose rows flag different frames does one pass, not
// two (rows flag a single frame almost always).  Frames not computed come
// back as 0 (the caller keeps their fast values).
__device__ __forceinline__ void tw_resolve(const MatParams& m, const uint32_t (&zh)[4], V3 wi, V3 wo,
                                           uint32_t (&x16)[6], uint32_t frames) {
  float raw[12];
  frame_raw_seq(m, zh, raw);
  float ti[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, to[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t todo = frames & (m.n_frames == 2 ? 3u : 1u);
  const uint32_t warp = __activemask();
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    if (!__any_sync(warp, todo != 0u)) break;
    const bool act = todo != 0u;
    const bool f1 = !(todo & 1u);  // this lane's next frame: 0 first
    float r6[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) r6[k] = f1 ? raw[6 + k] : raw[k];
    float a[3], b[3];
    frame_tw64_rsq(r6, d3(wi), d3(wo), a, b);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (act && !f1) { ti[k] = a[k]; to[k] = b[k]; }
      if (act && f1) { ti[3 + k] = a[k]; to[3 + k] = b[k]; }
    }
    todo &= f1 ? ~2u : ~1u;
  }
  pack_tw(m, ti, to, x16);
}

// fp16 halves of the 2-frame decoder direction words that belong to frame 0
// (the rest to frame 1): [t1.wi b1.wi | n1.wi t2.wi | b2.wi n2.wi | same for wo]
__device__ __forceinline__ uint32_t frame0_halves(int word) {
  return (word == 0 || word == 3) ? 0xFFFFFFFFu : ((word == 1 || word == 4) ? 0x0000FFFFu : 0u);
}

// Warp-cooperative re-evaluation of one query's BRDF decoder on the CUDA
// cores (fp32, the reference's fused_forward arithmetic up to summation
// order: mlp.py:196-208).  All 32 lanes call it with the same `src` lane;
// that lane holds the query's fp16 decoder input (in16: brdf_in values as
// packed pairs).  Lane j owns hidden units j and j + 32.  Returns the raw
// outputs y[0..out) on every lane.
__device__ __forceinline__ void brdf_simt_warp(const MatParams& m, const uint32_t (&in16)[10], int src,
                                               float (&y)[6]) {
  const int lane = threadIdx.x & 31;
  float h0 = 0.f, h1 = 0.f;  // this lane's activations (units lane, lane + 32)
  const int nl = m.brdf_count;
  for (int l = 0; l < nl; ++l) {
    const LayerDesc& L = m.layers[m.brdf_first + l];
    const int fi = L.fan_in, fo = L.out;
    const float* W = m.w32 + L.w32_off;  // [fo][fi + 1]
    const bool last = l == nl - 1;
    if (!last) {
      float a0 = 0.f, a1 = 0.f;
      const int j0 = lane, j1 = lane + 32;
      if (l == 0) {  // fan-in <= 20 (host-validated)
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          const float2 f = unpack_h2(__shfl_sync(0xffffffffu, in16[c], src));
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int k = 2 * c + e;
            const float xk = e ? f.y : f.x;
            if (k < fi) {
              if (j0 < fo) a0 = __fmaf_rn(xk, __ldg(W + (size_t)j0 * (fi + 1) + k), a0);
              if (j1 < fo) a1 = __fmaf_rn(xk, __ldg(W + (size_t)j1 * (fi + 1) + k), a1);
            }
          }
        }
      } else {
        for (int k = 0; k < fi; ++k) {
          const float xk = __shfl_sync(0xffffffffu, k < 32 ? h0 : h1, k & 31);
          if (j0 < fo) a0 = __fmaf_rn(xk, __ldg(W + (size_t)j0 * (fi + 1) + k), a0);
          if (j1 < fo) a1 = __fmaf_rn(xk, __ldg(W + (size_t)j1 * (fi + 1) + k), a1);
        }
      }
      if (j0 < fo) a0 += __ldg(W + (size_t)j0 * (fi + 1) + fi);
      if (j1 < fo) a1 += __ldg(W + (size_t)j1 * (fi + 1) + fi);
      if (L.act) {
        a0 = a0 >= 0.f ? a0 : kLeaky * a0;
        a1 = a1 >= 0.f ? a1 : kLeaky * a1;
      }
      h0 = j0 < fo ? a0 : 0.f;
      h1 = j1 < fo ? a1 : 0.f;
    } else {
#pragma unroll
      for (int o = 0; o < 6; ++o) {
        float p = 0.f;
        if (o < fo) {
          if (lane < fi) p = h0 * __ldg(W + (size_t)o * (fi + 1) + lane);
          if (lane + 32 < fi) p = __fmaf_rn(h1, __ldg(W + (size_t)o * (fi + 1) + lane + 32), p);
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) p += __shfl_xor_sync(0xffffffffu, p, d);
          p += __ldg(W + (size_t)o * (fi + 1) + fi);
        }
        y[o] = p;
      }
    }
  }
}

// Per-pixel sample mean in the eval epilogue (the renderer's spp
// accumulation, render.py:565): rows q = pixel * spp + s, spp = 2^spp_log2,
// consecutive rows on consecutive lanes.  The warp sums each aligned segment
// of min(spp, 32) lanes with shuffles and its first lane adds the segment's
// share of the mean to img[pixel] (fp32 atomics: 1 per 32 samples at spp >= 32).
// Warp-collective: every lane calls it (rows past the batch with valid = false).
__device__ __forceinline__ void spp_accumulate(float* img, int64_t q, V3 f, bool valid, int spp_log2) {
  const float inv = __int_as_float((127 - spp_log2) << 23);  // 2^-spp_log2, exact
  float x = valid ? f.x * inv : 0.f, y = valid ? f.y * inv : 0.f, z = valid ? f.z * inv : 0.f;
  const int seg = spp_log2 < 5 ? (1 << spp_log2) : 32;
  for (int d = seg >> 1; d > 0; d >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, d);
    y += __shfl_xor_sync(0xffffffffu, y, d);
    z += __shfl_xor_sync(0xffffffffu, z, d);
  }
  if (valid && ((threadIdx.x & 31) & (seg - 1)) == 0) {
    float* o = img + 3 * (q >> spp_log2);
    atomicAdd(o, x);
    atomicAdd(o + 1, y);
    atomicAdd(o + 2, z);
  }
}

}  // namespace dev
}  // namespace nmq
