// nmq_kl.cu — the per-row heads of the KL sampler loss (
// reference training.py:219-273 sampler_loss_and_grads and its default
// target training.py:187-216 _brdf_target_and_grad), around the fp32
// network engine of nmq_train.cu:
//
//   sampler forward_cached ([z, wi] -> raw)            nm_mlp_forward_cached
//   kl_sample_kernel: proxy from raw, one diffuse and one specular sample
//     per row (proxy.py:149-165), the BRDF decoder input at both samples
//   BRDF forward_cached on the 2B rows                 nm_mlp_forward_cached
//   kl_target_kernel: target lum(f) cos + eps and d target / d y
//   BRDF backward (input gradients)                    nm_mlp_backward
//   kl_target_dir_kernel: d target / d wo (frames adjoint, training.py:207-215)
//   kl_grad_kernel: grad log pdf (proxy.py:203-250), the sample Jacobians
//     (proxy.py:253-282), the raw-output Jacobian (neural.py:334-350) ->
//     per-row loss terms and d loss / d raw
//   sampler backward (parameter gradients)             nm_mlp_backward
//
// One thread per row, float64 like the reference (which runs these heads in
// numpy float64).  Every kernel is a few hundred FP64 flops per row over
// ~200 B of row state: latency/FP64 bound, tiny next to the MLP passes.
#include <cstdint>
#include <cuda_runtime.h>
#include "nmq_internal.h"

namespace nmq {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTiny = 1e-30;      // training.py:47 / proxy.py:35
constexpr double kEpsKL = 1e-4;      // training.py:45
constexpr double kAlphaFloor = 1e-4;  // proxy.py:32
constexpr int kMaxFrames = 4;

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 d3(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ double norm(D3 a) { return sqrt(dot(a, a)); }
__device__ __forceinline__ D3 ld3(const double* p) { return {p[0], p[1], p[2]}; }
__device__ __forceinline__ void st3(double* p, D3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }

// neural.py:46-64
__device__ __forceinline__ double quad_tanh(double x) {
  const double ax = fabs(x);
  const double v = x * (1.0 + 0.5 * ax) / (1.0 + ax + 0.5 * x * x);
  return fmin(fmax(v, -1.0), 1.0);
}
__device__ __forceinline__ double quad_tanh_grad(double x) {
  const double ax = fabs(x), den = 1.0 + ax + 0.5 * x * x;
  return (1.0 + ax) / (den * den);
}
__device__ __forceinline__ double quad_sinh(double x) { return x * (1.0 + x * x / 6.0); }
__device__ __forceinline__ double quad_sinh_grad(double x) { return 1.0 + 0.5 * x * x; }

// ProxyParams (proxy.py:37-84) from the raw sampler outputs (neural.py:317-331)
struct Prx {
  double wd, ws, mdx, mdy, ax, ay, rho, msx, msy, s;
};
__device__ Prx prx_from_raw(const float* raw, bool iso) {
  Prx p;
  if (iso) {
    p.wd = 0.5 * (quad_tanh((double)raw[0]) + 1.0);
    p.ws = 1.0 - p.wd;
    const double a = 0.5 * (quad_tanh((double)raw[1]) + 1.0);
    p.mdx = p.mdy = 0.0;
    p.ax = p.ay = a;
    p.rho = 0.0;
    p.msx = p.msy = 0.0;
  } else {
    const double a = raw[0], b = raw[3], m = fmax(a, b);  // softmax_pair (neural.py:67-71)
    const double ea = exp(a - m), eb = exp(b - m);
    p.wd = ea / (ea + eb);
    p.ws = eb / (ea + eb);
    p.mdx = quad_sinh((double)raw[1]);
    p.mdy = quad_sinh((double)raw[2]);
    p.ax = 0.5 * (quad_tanh((double)raw[4]) + 1.0);
    p.ay = 0.5 * (quad_tanh((double)raw[5]) + 1.0);
    p.rho = quad_tanh((double)raw[6]);
    p.msx = quad_sinh((double)raw[7]);
    p.msy = quad_sinh((double)raw[8]);
  }
  p.ax = fmax(p.ax, kAlphaFloor);
  p.ay = fmax(p.ay, kAlphaFloor);
  const double rc = sqrt(1.0 - 1e-4);
  p.rho = fmin(fmax(p.rho, -rc), rc);
  p.s = sqrt(1.0 - p.rho * p.rho);
  return p;
}
__device__ __forceinline__ D3 diffuse_normal(const Prx& p) {  // proxy.py:80-84 (no floor)
  const D3 v = d3(-p.mdx, -p.mdy, 1.0);
  return (1.0 / norm(v)) * v;
}

// Orthonormal frames from the frame layer's raw outputs (neural.py:207-233,
// geom.py:82-89 fallback tangent)
struct Fr {
  D3 t, b, n;
};
__device__ Fr frame_from_raw(const float* r) {
  const D3 rn = d3(r[0], r[1], r[2]);
  D3 rt = d3(r[3], r[4], r[5]);
  const D3 n = (1.0 / fmax(norm(rn), 1e-12)) * rn;
  D3 c = cross(n, rt);
  double cl = norm(c);
  if (cl < 1e-8) {
    const double ax = fabs(n.x), ay = fabs(n.y), az = fabs(n.z);
    const int k = (ax <= ay && ax <= az) ? 0 : (ay <= az ? 1 : 2);  // argmin, first on ties
    const D3 e = d3(k == 0, k == 1, k == 2);
    const D3 ce = cross(n, e);
    rt = (1.0 / norm(ce)) * ce;
    c = cross(n, rt);
    cl = norm(c);
  }
  const D3 b = (1.0 / fmax(cl, 1e-12)) * c;
  return {cross(b, n), b, n};
}

// uniform sphere (geom.py:121-126) and unit-roughness NDF (proxy.py:138-146)
__device__ __forceinline__ D3 uniform_sphere(double u0, double u1) {
  const double z = 1.0 - 2.0 * u0, r = sqrt(fmax(0.0, 1.0 - z * z)), phi = 2.0 * kPi * u1;
  return d3(r * cos(phi), r * sin(phi), z);
}
__device__ __forceinline__ D3 ndf_sample(double u0, double u1) {
  const double tan2 = u0 / fmax(1.0 - u0, 1e-12);
  const double ct = 1.0 / sqrt(1.0 + tan2), st = sqrt(fmax(0.0, 1.0 - ct * ct));
  const double phi = 2.0 * kPi * u1;
  return d3(st * cos(phi), st * sin(phi), ct);
}
__device__ __forceinline__ D3 warp_m(const Prx& p, D3 m) {  // M m (proxy.py:62-73)
  return d3(p.ax * m.x - p.msx * m.z, p.ay * p.rho * m.x + p.ay * p.s * m.y - p.msy * m.z, m.z);
}

// scratch row layout (doubles)
enum { kWoD = 0, kWoS = 3, kGlD = 6, kV = 7, kM = 10, kH = 13, kGlS = 16, kScr = 17 };

// decoder input [z, T wi, T wo] (frames) or [z, wi, wo] (neural.py:261-270), as fp32
__device__ void decoder_row(float* x, const float* z, const Fr* fr, int nf, bool frames, D3 wi, D3 wo) {
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = z[c];
  if (!frames) {
    x[8] = (float)wi.x; x[9] = (float)wi.y; x[10] = (float)wi.z;
    x[11] = (float)wo.x; x[12] = (float)wo.y; x[13] = (float)wo.z;
    return;
  }
  for (int f = 0; f < nf; ++f) {
    x[8 + 3 * f] = (float)dot(fr[f].t, wi);
    x[9 + 3 * f] = (float)dot(fr[f].b, wi);
    x[10 + 3 * f] = (float)dot(fr[f].n, wi);
    x[8 + 3 * nf + 3 * f] = (float)dot(fr[f].t, wo);
    x[9 + 3 * nf + 3 * f] = (float)dot(fr[f].b, wo);
    x[10 + 3 * nf + 3 * f] = (float)dot(fr[f].n, wo);
  }
}

__global__ void kl_sample_kernel(int64_t b, int frames, int nf, int iso, int rs,
                                 const float* __restrict__ raw_s, const float* __restrict__ raw_f,
                                 const float* __restrict__ z, const double* __restrict__ wi,
                                 const double* __restrict__ u_d, const double* __restrict__ u_s,
                                 float* __restrict__ x2, double* __restrict__ scr) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= b) return;
  const Prx p = prx_from_raw(raw_s + i * rs, iso);
  const D3 w = ld3(wi + 3 * i);
  double* s = scr + i * kScr;
  // diffuse (proxy.py:149-156): offset-sphere construction
  const D3 v = uniform_sphere(u_d[2 * i], u_d[2 * i + 1]);
  const D3 g = diffuse_normal(p) + v;
  const double gl = fmax(norm(g), 1e-9);
  const D3 wo_d = (1.0 / gl) * g;
  // specular (proxy.py:159-165)
  const D3 m = ndf_sample(u_s[2 * i], u_s[2 * i + 1]);
  const D3 gs = warp_m(p, m);
  const double gls = norm(gs);
  const D3 h = (1.0 / fmax(gls, 1e-12)) * gs;
  const D3 wo_s = (2.0 * dot(w, h)) * h - w;  // geom.reflect
  st3(s + kWoD, wo_d);
  st3(s + kWoS, wo_s);
  s[kGlD] = gl;
  st3(s + kV, v);
  st3(s + kM, m);
  st3(s + kH, h);
  s[kGlS] = gls;
  Fr fr[kMaxFrames];
  if (frames)
    for (int f = 0; f < nf; ++f) fr[f] = frame_from_raw(raw_f + i * 6 * nf + 6 * f);
  const int in_w = frames ? 8 + 6 * nf : 14;
  decoder_row(x2 + i * in_w, z + 8 * i, fr, nf, frames, w, wo_d);
  decoder_row(x2 + (b + i) * in_w, z + 8 * i, fr, nf, frames, w, wo_s);
}

// rows [0, b): diffuse samples, [b, 2b): specular samples
__global__ void kl_target_kernel(int64_t b, int out_w, const float* __restrict__ y,
                                 const double* __restrict__ scr, double* __restrict__ tgt,
                                 double* __restrict__ lum, float* __restrict__ og) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= 2 * b) return;
  const int64_t i = r < b ? r : r - b;
  const double woz_raw = scr[i * kScr + (r < b ? kWoD : kWoS) + 2];
  const bool up = woz_raw > 0.0;
  const double woz = fmax(woz_raw, 0.0);
  const double lw[3] = {0.2126, 0.7152, 0.0722};  // training.py:46
  double l = 0.0;
  for (int k = 0; k < out_w; ++k) {
    const double yk = y[r * out_w + k];
    if (k < 3) {
      l += lw[k] * fmax(expm1(fmin(yk, 60.0)), 0.0);                           // brdf_output
      og[r * out_w + k] = (float)(lw[k] * (yk > 0.0 ? exp(fmin(yk, 60.0)) : 0.0) * woz);  // ..._grad
    } else {
      og[r * out_w + k] = 0.f;
    }
  }
  lum[r] = l;
  tgt[r] = (up ? l * woz : 0.0) + kEpsKL;
}

// d target / d wo: the wo block of the decoder-input gradient through the
// frames' transform adjoint (neural.py:198-205), + lum e_z, zero below the horizon
__global__ void kl_target_dir_kernel(int64_t b, int frames, int nf, const float* __restrict__ raw_f,
                                     const double* __restrict__ dx, const double* __restrict__ scr,
                                     const double* __restrict__ lum, double* __restrict__ dtgt) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= 2 * b) return;
  const int64_t i = r < b ? r : r - b;
  const int in_w = frames ? 8 + 6 * nf : 14;
  const double* g = dx + r * in_w;
  D3 d;
  if (frames) {
    d = d3(0, 0, 0);
    for (int f = 0; f < nf; ++f) {
      const Fr fr = frame_from_raw(raw_f + i * 6 * nf + 6 * f);
      const double* gf = g + 8 + 3 * nf + 3 * f;
      d = d + (gf[0] * fr.t + gf[1] * fr.b + gf[2] * fr.n);
    }
  } else {
    d = d3(g[11], g[12], g[13]);
  }
  d.z += lum[r];
  const bool up = scr[i * kScr + (r < b ? kWoD : kWoS) + 2] > 0.0;
  st3(dtgt + 3 * r, up ? d : d3(0, 0, 0));
}

// (p, d log p / d wo) of the mixture at wo (proxy.py:203-250)
__device__ double grad_log_pdf(const Prx& p, D3 wi, D3 wo, D3& dlogp) {
  const D3 nd = diffuse_normal(p);
  const double dn = dot(wo, nd);
  const double pd = fmax(dn, 0.0) / kPi;
  const D3 dpd = dn > 0.0 ? (1.0 / kPi) * nd : d3(0, 0, 0);
  D3 h = wi + wo;  // _half_vectors (proxy.py:87-101)
  const double hl = norm(h);
  const bool ok = hl > 1e-9;
  h = (1.0 / fmax(hl, 1e-12)) * h;
  const double flip = h.z < 0.0 ? -1.0 : 1.0;
  h = flip * h;
  const bool hz_ok = ok && h.z > 0.0;
  const double qx = (h.x + p.msx * h.z) / p.ax;  // _q_vector (proxy.py:104-111)
  const double qy = ((h.y + p.msy * h.z) / p.ay - p.rho * qx) / p.s;
  const D3 q = d3(qx, qy, h.z);
  const double qn2 = fmax(dot(q, q), kTiny);
  const double coh = dot(wo, h);
  const double det = p.ax * p.ay * p.s;
  double ps = 0.0;
  D3 dps = d3(0, 0, 0);
  if (hz_ok) {
    ps = h.z / (det * 4.0 * kPi * qn2 * qn2 * fmax(fabs(coh), 1e-12));
    const D3 mtq = d3(q.x / p.ax - q.y * p.rho / (p.ax * p.s), q.y / (p.ay * p.s),
                      q.x * p.msx / p.ax + q.y * (p.msy / (p.ay * p.s) - p.msx * p.rho / (p.ax * p.s)) + q.z);
    const double inv_coh = fabs(coh) < 1e-12 ? 0.0 : 1.0 / coh;
    const D3 dlog_dh = d3(0, 0, 1.0 / fmax(h.z, 1e-12)) - (4.0 / qn2) * mtq - inv_coh * wo;
    const double wsl = fmax(norm(wi + wo), 1e-12);
    const D3 proj = dlog_dh - dot(h, dlog_dh) * h;
    dps = ps * ((flip / wsl) * proj - inv_coh * h);
  }
  const double pm = p.wd * pd + p.ws * ps;
  const D3 dp = p.wd * dpd + p.ws * dps;
  dlogp = (1.0 / fmax(pm, kTiny)) * dp;
  return pm;
}

__global__ void kl_grad_kernel(int64_t b, int iso, int rs, const float* __restrict__ raw_s,
                               const double* __restrict__ wi, const double* __restrict__ scr,
                               const double* __restrict__ tgt, const double* __restrict__ dtgt,
                               float* __restrict__ draw, double* __restrict__ loss_rows) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= b) return;
  const float* raw = raw_s + i * rs;
  const Prx p = prx_from_raw(raw, iso);
  const D3 w = ld3(wi + 3 * i);
  const double* s = scr + i * kScr;
  const D3 wo_d = ld3(s + kWoD), wo_s = ld3(s + kWoS);
  D3 dl_d, dl_s;
  const double p_d = grad_log_pdf(p, w, wo_d, dl_d);
  const double p_s = grad_log_pdf(p, w, wo_s, dl_s);
  const double f_d = tgt[i], f_s = tgt[b + i];
  const double ell_d = log(fmax(p_d, kTiny)) - log(f_d);
  const double ell_s = log(fmax(p_s, kTiny)) - log(f_s);
  loss_rows[i] = p.wd * ell_d + p.ws * ell_s;
  const D3 brk_d = dl_d - (1.0 / f_d) * ld3(dtgt + 3 * i);
  const D3 brk_s = dl_s - (1.0 / f_s) * ld3(dtgt + 3 * (b + i));
  // diffuse Jacobian d wo / d mu_d (proxy.py:253-266)
  const D3 nd = diffuse_normal(p);
  const double vlen = sqrt(1.0 + p.mdx * p.mdx + p.mdy * p.mdy);
  const double gl = s[kGlD];
  double g_mu_d[2];
  for (int k = 0; k < 2; ++k) {
    const D3 e = d3(k == 0 ? -1.0 : 0.0, k == 1 ? -1.0 : 0.0, 0.0);
    const D3 dnd = (1.0 / vlen) * (e - dot(nd, e) * nd);
    const D3 dwo = (1.0 / gl) * (dnd - dot(wo_d, dnd) * wo_d);
    g_mu_d[k] = p.wd * dot(brk_d, dwo);
  }
  // specular Jacobian d wo / d (ax, ay, rho, msx, msy) (proxy.py:269-282)
  const D3 m = ld3(s + kM), h = ld3(s + kH);
  const double gls = s[kGlS];
  const D3 dg[5] = {d3(m.x, 0, 0), d3(0, p.rho * m.x + p.s * m.y, 0),
                    d3(0, p.ay * (m.x - p.rho * m.y / p.s), 0), d3(-m.z, 0, 0), d3(0, -m.z, 0)};
  const double wih = dot(w, h);
  double g_spec[5];
  for (int k = 0; k < 5; ++k) {
    const D3 dh = (1.0 / gls) * (dg[k] - dot(h, dg[k]) * h);
    const D3 dwo = (2.0 * dot(w, dh)) * h + (2.0 * wih) * dh;
    g_spec[k] = p.ws * dot(brk_s, dwo);
  }
  // raw-output Jacobian (neural.py:334-350), / b for the batch mean
  const double ib = 1.0 / (double)b;
  float* d = draw + i * rs;
  if (iso) {
    d[0] = (float)((ell_d - ell_s) * 0.5 * quad_tanh_grad((double)raw[0]) * ib);
    d[1] = (float)((g_spec[0] + g_spec[1]) * 0.5 * quad_tanh_grad((double)raw[1]) * ib);
  } else {
    const double a = raw[0], bb = raw[3], mx = fmax(a, bb);
    const double ea = exp(a - mx), eb = exp(bb - mx);
    const double sj = (ea / (ea + eb)) * (eb / (ea + eb));
    d[0] = (float)((ell_d - ell_s) * sj * ib);
    d[3] = (float)((ell_s - ell_d) * sj * ib);
    d[1] = (float)(g_mu_d[0] * quad_sinh_grad((double)raw[1]) * ib);
    d[2] = (float)(g_mu_d[1] * quad_sinh_grad((double)raw[2]) * ib);
    d[4] = (float)(g_spec[0] * 0.5 * quad_tanh_grad((double)raw[4]) * ib);
    d[5] = (float)(g_spec[1] * 0.5 * quad_tanh_grad((double)raw[5]) * ib);
    d[6] = (float)(g_spec[2] * quad_tanh_grad((double)raw[6]) * ib);
    d[7] = (float)(g_spec[3] * quad_sinh_grad((double)raw[7]) * ib);
    d[8] = (float)(g_spec[4] * quad_sinh_grad((double)raw[8]) * ib);
  }
}

inline unsigned grid_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t launch_kl_sample(int64_t b, int frames, int nf, int iso, const float* raw_s,
                             const float* raw_f, const float* z, const double* wi, const double* u_d,
                             const double* u_s, float* x2, double* scr, cudaStream_t st) {
  if (nf > kMaxFrames) return cudaErrorInvalidValue;
  kl_sample_kernel<<<grid_for(b), 256, 0, st>>>(b, frames, nf, iso, iso ? 2 : 9, raw_s, raw_f, z, wi,
                                                u_d, u_s, x2, scr);
  return cudaGetLastError();
}
cudaError_t launch_kl_target(int64_t b, int out_w, const float* y, const double* scr, double* tgt,
                             double* lum, float* og, cudaStream_t st) {
  kl_target_kernel<<<grid_for(2 * b), 256, 0, st>>>(b, out_w, y, scr, tgt, lum, og);
  return cudaGetLastError();
}
cudaError_t launch_kl_target_dir(int64_t b, int frames, int nf, const float* raw_f, const double* dx,
                                 const double* scr, const double* lum, double* dtgt, cudaStream_t st) {
  if (nf > kMaxFrames) return cudaErrorInvalidValue;
  kl_target_dir_kernel<<<grid_for(2 * b), 256, 0, st>>>(b, frames, nf, raw_f, dx, scr, lum, dtgt);
  return cudaGetLastError();
}
cudaError_t launch_kl_grad(int64_t b, int iso, const float* raw_s, const double* wi, const double* scr,
                           const double* tgt, const double* dtgt, float* draw, double* loss_rows,
                           cudaStream_t st) {
  kl_grad_kernel<<<grid_for(b), 256, 0, st>>>(b, iso, iso ? 2 : 9, raw_s, wi, scr, tgt, dtgt, draw,
                                              loss_rows);
  return cudaGetLastError();
}

}  // namespace nmq
