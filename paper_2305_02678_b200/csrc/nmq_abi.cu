// nmq_abi.cu — C ABI (include/nmq.h): material creation (re-tiling the
// reference's packed fp16 weights into the UMMA B-operand layout, latent
// upload) and the query entry points.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <thread>
#include <cstdio>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <cuda_fp16.h>
#include "../../include/nmq.h"
#include "nmq_internal.h"

using namespace nmq;

namespace {

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(NM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

// Write B operand of one layer into `blob` (fp16 bits) at byte offset `off`.
// Layout: chunk-major K-major, chunk c (8 K values) of row n at
//   off + c*(n_pad*16) + n*16.
struct Packer {
  std::vector<uint16_t> blob;  // fp16 bits
  uint32_t append(int n_pad, int k_chunks) {
    const uint32_t off = (uint32_t)(blob.size() * 2);
    blob.resize(blob.size() + (size_t)n_pad * k_chunks * 8, 0);
    return off;
  }
  void set(uint32_t off, int n_pad, int n, int k, uint16_t v) {
    const int c = k / 8, e = k % 8;
    blob[off / 2 + (size_t)c * n_pad * 8 + (size_t)n * 8 + e] = v;
  }
};

struct NetView {
  int n_layers;
  std::vector<int> fi, fo, act;
  std::vector<size_t> ofs;  // offset of each layer in the packed array (halves)
  const uint16_t* packed;
  const float* weights;     // fp32 master weights (same order) or null
};

// fp32 -> (hi, lo) fp16 bits with hi + lo = v to ~2^-22 (clamped to fp16 range)
void split_f32(float v, uint16_t& hi, uint16_t& lo) {
  const float c = v > 65504.f ? 65504.f : (v < -65504.f ? -65504.f : v);
  const __half h = __float2half_rn(c);
  const __half l = __float2half_rn(c - __half2float(h));
  hi = *reinterpret_cast<const uint16_t*>(&h);
  lo = *reinterpret_cast<const uint16_t*>(&l);
}

int view_net(const nm_net_desc& d, const char* name, NetView& v) {
  if (d.n_layers <= 0 || !d.fan_in || !d.fan_out || !d.act || !d.packed)
    return fail(NM_ERR_INVALID, std::string(name) + ": empty network description");
  v.n_layers = d.n_layers;
  v.packed = d.packed;
  v.weights = d.weights;
  size_t o = 0;
  for (int l = 0; l < d.n_layers; ++l) {
    v.fi.push_back(d.fan_in[l]);
    v.fo.push_back(d.fan_out[l]);
    v.act.push_back(d.act[l]);
    v.ofs.push_back(o);
    if (d.fan_in[l] <= 0 || d.fan_out[l] <= 0)
      return fail(NM_ERR_INVALID, std::string(name) + ": bad layer size");
    if (l > 0 && d.fan_in[l] != d.fan_out[l - 1])
      return fail(NM_ERR_INVALID, "layer dimensions do not chain");  // mlp.py:53-55
    if (d.act[l] != NM_ACT_LINEAR && d.act[l] != NM_ACT_LEAKY)
      return fail(NM_ERR_INVALID, "unknown activation code");
    o += (size_t)d.fan_out[l] * (d.fan_in[l] + 1);
  }
  return NM_OK;
}

// Pack one chain of layers.  The first layer takes an input vector with its
// bias slot at index fan_in; later layers take the hi/lo split of the
// previous padded activation plus the shared bias chunk.
float h2f(uint16_t bits) {
  __half_raw r;
  r.x = bits;
  return __half2float(__half(r));
}

// fp32 copy of one network in the reference's packed access order (the
// fp16 weights widened exactly, or the fp32 master weights for `precise`).
void append_w32(const NetView& v, bool precise, std::vector<float>& w32, MatParams& mp, int first) {
  for (int l = 0; l < v.n_layers; ++l) {
    LayerDesc& L = mp.layers[first + l];
    L.fan_in = (uint16_t)v.fi[l];
    L.w32_off = (uint32_t)w32.size();
    const size_t cnt = (size_t)v.fo[l] * (v.fi[l] + 1);
    for (size_t i = 0; i < cnt; ++i)
      w32.push_back(precise ? v.weights[v.ofs[l] + i] : h2f(v.packed[v.ofs[l] + i]));
  }
}

int pack_chain(const NetView& v, Packer& pk, MatParams& mp, int& n_layers, const char* name) {
  if (mp.precise) {
    // fp32 path: B = [W_hi | W_hi | W_lo] (+ bias chunk [b_hi, 0, b_lo, 0 ...]
    // for hidden-input layers, against the A bias chunk (1, 0, 1, 0 ...))
    if (!v.weights) return fail(NM_ERR_INVALID, std::string(name) + ": precise material needs fp32 weights");
    for (int l = 0; l < v.n_layers; ++l) {
      if (n_layers >= kMaxLayers) return fail(NM_ERR_UNSUPPORTED, "too many layers");
      LayerDesc L{};
      const int fi = v.fi[l], fo = v.fo[l];
      const int n_pad = round_up(fo, 16);
      if (n_pad > kMaxWidth)
        return fail(NM_ERR_UNSUPPORTED, std::string(name) + ": layer width > 64 not supported");
      L.n_pad = (uint16_t)n_pad;
      L.out = (uint8_t)fo;
      L.act = (uint8_t)v.act[l];
      L.precise = 1;
      const float* w = v.weights + v.ofs[l];  // [fo][fi+1]
      auto put3 = [&](uint32_t off, int kp, int n, int k, float val) {
        uint16_t hi, lo;
        split_f32(val, hi, lo);
        pk.set(off, n_pad, n, k, hi);
        pk.set(off, n_pad, n, kp + k, hi);
        pk.set(off, n_pad, n, 2 * kp + k, lo);
      };
      if (l == 0) {
        const int k_pad = round_up(fi + 1, 16);
        if (k_pad > 32) return fail(NM_ERR_UNSUPPORTED, std::string(name) + ": input too wide");
        L.first = 1;
        L.ksteps = (uint8_t)(k_pad / 16);
        L.b_off = pk.append(n_pad, 3 * k_pad / 8);
        if (k_pad > mp.dmax) mp.dmax = k_pad;  // A holds x_hi and x_lo: k_pad columns
        for (int n = 0; n < fo; ++n)
          for (int k = 0; k <= fi; ++k) put3(L.b_off, k_pad, n, k, w[(size_t)n * (fi + 1) + k]);
      } else {
        const int in_pad = round_up(fi, 16);
        L.first = 0;
        L.in_pad = (uint16_t)in_pad;
        L.ksteps = (uint8_t)(3 * in_pad / 16 + 1);
        L.b_off = pk.append(n_pad, 3 * in_pad / 8 + 2);
        for (int n = 0; n < fo; ++n) {
          for (int k = 0; k < fi; ++k) put3(L.b_off, in_pad, n, k, w[(size_t)n * (fi + 1) + k]);
          uint16_t bh, bl;
          split_f32(w[(size_t)n * (fi + 1) + fi], bh, bl);
          pk.set(L.b_off, n_pad, n, 3 * in_pad, bh);
          pk.set(L.b_off, n_pad, n, 3 * in_pad + 2, bl);
        }
      }
      if ((int)L.n_pad > mp.dmax) mp.dmax = L.n_pad;
      mp.layers[n_layers++] = L;
    }
    return NM_OK;
  }
  for (int l = 0; l < v.n_layers; ++l) {
    if (n_layers >= kMaxLayers) return fail(NM_ERR_UNSUPPORTED, "too many layers");
    LayerDesc L{};
    const int fi = v.fi[l], fo = v.fo[l];
    const int n_pad = round_up(fo, 16);
    if (n_pad > kMaxWidth)
      return fail(NM_ERR_UNSUPPORTED, std::string(name) + ": layer width > 64 not supported");
    L.n_pad = (uint16_t)n_pad;
    L.out = (uint8_t)fo;
    L.act = (uint8_t)v.act[l];
    const uint16_t* w = v.packed + v.ofs[l];  // [fo][fi+1]
    if (l == 0) {
      const int k_pad = round_up(fi + 1, 16);
      if (k_pad > 32) return fail(NM_ERR_UNSUPPORTED, std::string(name) + ": input too wide");
      L.first = 1;
      L.in_pad = 0;
      L.ksteps = (uint8_t)(k_pad / 16);
      L.b_off = pk.append(n_pad, k_pad / 8);
      for (int n = 0; n < fo; ++n) {
        for (int k = 0; k < fi; ++k) pk.set(L.b_off, n_pad, n, k, w[(size_t)n * (fi + 1) + k]);
        pk.set(L.b_off, n_pad, n, fi, w[(size_t)n * (fi + 1) + fi]);  // bias vs x[fi] = 1
      }
    } else {
      const int in_pad = round_up(fi, 16);
      L.first = 0;
      L.in_pad = (uint16_t)in_pad;
      L.ksteps = (uint8_t)(2 * in_pad / 16 + 1);
      const int k_chunks = 2 * in_pad / 8 + 2;
      L.b_off = pk.append(n_pad, k_chunks);
      for (int n = 0; n < fo; ++n) {
        for (int k = 0; k < fi; ++k) {
          const uint16_t wv = w[(size_t)n * (fi + 1) + k];
          pk.set(L.b_off, n_pad, n, k, wv);           // against hi
          pk.set(L.b_off, n_pad, n, in_pad + k, wv);  // against lo
        }
        // bias twice: the A-side bias chunk holds (beta_hi, beta_lo) so the
        // MMA adds beta * b exactly (beta = 1 generic, c^depth fast path)
        const uint16_t bv = w[(size_t)n * (fi + 1) + fi];
        pk.set(L.b_off, n_pad, n, 2 * in_pad, bv);
        pk.set(L.b_off, n_pad, n, 2 * in_pad + 1, bv);
      }
    }
    if ((int)L.n_pad > mp.dmax) mp.dmax = L.n_pad;
    mp.layers[n_layers++] = L;
  }
  return NM_OK;
}

// Does the material match one of the specialized pipelined kernels
// (nmq_fast.cu)?  All of them: 2 learned frames, 3x32 sampler (9 outputs or
// isotropic 2), leaky hidden layers, linear outputs, equal hidden widths.
int detect_fast_arch(const MatParams& mp, const NetView& bv, const NetView& sv,
                     const nm_material_desc* d) {
  if (!mp.has_brdf || !mp.has_sampler || !d->use_frames || d->n_frames != 2) return -1;
  auto uniform = [](const NetView& v, int w) {
    for (int l = 0; l < v.n_layers; ++l) {
      const bool last = l == v.n_layers - 1;
      if (v.act[l] != (last ? NM_ACT_LINEAR : NM_ACT_LEAKY)) return false;
      if (!last && v.fo[l] != w) return false;
    }
    return true;
  };
  if (sv.n_layers != 4 || !uniform(sv, 32)) return -1;
  if (bv.n_layers == 3 && uniform(bv, 32)) return 0;
  if (bv.n_layers == 3 && uniform(bv, 16)) return 1;
  if (bv.n_layers == 4 && uniform(bv, 64)) return 2;
  return -1;
}

// Layers of the specialized kernels (see MatParams::fast_frame_off):
// re-packed frame layer and BRDF first layer for the shared input chunks,
// fp32 copy of the BRDF output layer for the FFMA2 path.
void fill_fast_layers(MatParams& mp, Packer& pk, const NetView& fv, const NetView& bv) {
  {
    const uint16_t* w = fv.packed + fv.ofs[0];  // [12][8 + 1]
    mp.fast_frame_off = pk.append(16, 2);
    for (int n = 0; n < 12; ++n) {
      for (int k = 0; k < 8; ++k) pk.set(mp.fast_frame_off, 16, n, k, w[n * 9 + k]);
      pk.set(mp.fast_frame_off, 16, n, 11, w[n * 9 + 8]);
    }
  }
  {
    const int fi = bv.fi[0], fo = bv.fo[0];  // 20 = [z(8), T.wi(6), T.wo(6)]
    const int n_pad = round_up(fo, 16);
    const uint16_t* w = bv.packed + bv.ofs[0];  // [fo][fi + 1]
    mp.fast_l1_off = pk.append(n_pad, 4);
    for (int n = 0; n < fo; ++n) {
      for (int k = 0; k < 8; ++k) pk.set(mp.fast_l1_off, n_pad, n, k, w[n * (fi + 1) + k]);
      for (int k = 8; k < 20; ++k) pk.set(mp.fast_l1_off, n_pad, n, k + 8, w[n * (fi + 1) + k]);
      pk.set(mp.fast_l1_off, n_pad, n, 11, w[n * (fi + 1) + fi]);
    }
  }
  const int l = bv.n_layers - 1;
  const int fi = bv.fi[l], fo = bv.fo[l];
  const uint16_t* w = bv.packed + bv.ofs[l];  // [fo][fi + 1]
  for (int j = 0; j < 6; ++j) {
    for (int q = 0; q < 32; ++q) {
      const int k0 = 2 * q, k1 = 2 * q + 1;
      const float a = (j < fo && k0 < fi) ? h2f(w[j * (fi + 1) + k0]) : 0.f;
      const float b = (j < fo && k1 < fi) ? h2f(w[j * (fi + 1) + k1]) : 0.f;
      mp.ow[j][q] = make_float2(a, b);
    }
    mp.ob[j] = j < fo ? h2f(w[j * (fi + 1) + fi]) : 0.f;
  }
}

}  // namespace

struct nm_mlp {
  int device = 0;
  int n_layers = 0;
  int32_t fi[kMaxLayers] = {}, fo[kMaxLayers] = {}, act[kMaxLayers] = {};
  int32_t w_floats = 0;
  float* w = nullptr;  // fp32 master weights, access order [w_row, bias] per neuron
};

struct nm_material {
  int device = 0;
  MatParams mp{};
  void* latent = nullptr;
  void* wblob = nullptr;
  void* w32 = nullptr;
  int64_t texels = 0;
  int brdf_width = 0, sampler_width = 0;
};

namespace {
// DIVERGENT's device table of the materials' parameter blocks, uploaded once
// per material list (handles are immutable) so a call never waits for the
// stream; entries holding a material are dropped when it is destroyed.
struct DivTable {
  int device;
  std::vector<const nm_material*> mats;
  nmq::MatParams* dev;
};
std::mutex g_div_mu;
std::vector<DivTable> g_div;

cudaError_t div_table(const std::vector<const nmq::MatParams*>& mps, const nm_material* const* mats, int32_t n_mats,
                      int device, nmq::MatParams** out) {
  std::lock_guard<std::mutex> lock(g_div_mu);
  std::vector<const nm_material*> key(mats, mats + n_mats);
  for (const DivTable& t : g_div)
    if (t.device == device && t.mats == key) {
      *out = t.dev;
      return cudaSuccess;
    }
  std::vector<nmq::MatParams> host(n_mats);
  for (int k = 0; k < n_mats; ++k) host[k] = *mps[k];
  nmq::MatParams* d = nullptr;
  cudaError_t e = cudaMalloc(&d, n_mats * sizeof(nmq::MatParams));
  if (e != cudaSuccess) return e;
  if ((e = cudaMemcpy(d, host.data(), n_mats * sizeof(nmq::MatParams), cudaMemcpyHostToDevice)) != cudaSuccess) {
    cudaFree(d);
    return e;
  }
  g_div.push_back({device, key, d});
  *out = d;
  return cudaSuccess;
}

void div_forget(const nm_material* m) {
  std::lock_guard<std::mutex> lock(g_div_mu);
  for (size_t i = 0; i < g_div.size();) {
    const auto& v = g_div[i].mats;
    if (std::find(v.begin(), v.end(), m) != v.end()) {
      cudaFree(g_div[i].dev);
      g_div.erase(g_div.begin() + i);
    } else {
      ++i;
    }
  }
}
}  // namespace

extern "C" {

const char* nm_last_error(void) { return t_err.c_str(); }
int nm_version(void) { return NMQ_VERSION; }
int64_t nm_launch_count(void) { return g_launches.load(); }
int nm_last_kernel_path(void) { return g_last_path.load(); }
int nm_set_tw_margin(float delta) {
  g_tw_margin = delta;
  return NM_OK;
}
int nm_set_kernel_path(int path) {
  if (path < 0 || path > 2) return fail(NM_ERR_INVALID, "kernel path must be 0..2");
  g_kernel_path = path;
  return NM_OK;
}

int nm_material_create(const nm_material_desc* d, int device, nm_material** out) {
  if (!d || !out) return fail(NM_ERR_INVALID, "null argument");
  *out = nullptr;
  if (d->channels != 8)
    return fail(NM_ERR_UNSUPPORTED, "latent channels must be 8 (one 16-byte texel)");
  if (d->width <= 0 || d->height <= 0) return fail(NM_ERR_INVALID, "bad latent size");
  // level chain, latent.py:28-38
  std::vector<LevelDesc> lv;
  {
    int w = d->width, h = d->height;
    int64_t off = 0;
    while (true) {
      lv.push_back(LevelDesc{w, h, off});
      off += (int64_t)w * h;
      if (w == 1 && h == 1) break;
      w = w / 2 > 1 ? w / 2 : 1;
      h = h / 2 > 1 ? h / 2 : 1;
    }
  }
  if ((int)lv.size() != d->n_levels)
    return fail(NM_ERR_INVALID, "corrupt pyramid header");  // latent.py:170-171
  if ((int)lv.size() > kMaxLevels) return fail(NM_ERR_UNSUPPORTED, "too many levels");
  const int64_t texel_bytes = d->latent_fp32 ? 32 : 16;
  if (!d->latent) return fail(NM_ERR_INVALID, "material has no latent pyramid");

  nm_material* m = new nm_material();
  m->device = device;
  MatParams& mp = m->mp;
  mp.n_levels = (int)lv.size();
  bool pow2 = true;
  for (size_t i = 0; i < lv.size(); ++i) {
    mp.lv[i] = lv[i];
    pow2 &= (lv[i].w & (lv[i].w - 1)) == 0 && (lv[i].h & (lv[i].h - 1)) == 0;
  }
  mp.pow2 = pow2 ? 1 : 0;
  mp.texel_fp32 = d->latent_fp32 ? 1 : 0;
  m->texels = lv.back().off + 1;

  // --- networks ---------------------------------------------------------------
  Packer pk;
  std::vector<float> w32;
  int nl = 0;
  mp.use_frames = d->use_frames ? 1 : 0;
  mp.n_frames = d->use_frames ? d->n_frames : 0;
  mp.albedo = d->albedo_head ? 1 : 0;
  mp.isotropic = d->sampler_isotropic ? 1 : 0;
  mp.precise = d->precise ? 1 : 0;
  mp.frame_layer = -1;
  int rc;
  NetView fv, bv, sv;
  if (d->use_frames && d->frame.n_layers > 0) {
    if (d->n_frames < 1 || d->n_frames > 2) {
      delete m;
      return fail(NM_ERR_UNSUPPORTED, "n_frames must be 1 or 2");
    }
    if ((rc = view_net(d->frame, "frame layer", fv)) != NM_OK) { delete m; return rc; }
    if (fv.n_layers != 1 || fv.fi[0] != 8 || fv.fo[0] != 6 * d->n_frames) {
      delete m;
      return fail(NM_ERR_INVALID, "frame layer must be one 8 -> 6*n_frames layer");
    }
    mp.frame_layer = nl;
    if ((rc = pack_chain(fv, pk, mp, nl, "frame layer")) != NM_OK) { delete m; return rc; }
    append_w32(fv, mp.precise, w32, mp, mp.frame_layer);
    // frame layer [W | b] in fp32 for the sequential-FMA evaluation (mlp.py:207)
    for (int n = 0; n < 6; ++n)
      for (int k = 0; k <= 8; ++k) {
        const size_t o = mp.layers[mp.frame_layer].w32_off;
        mp.fw2[n][k] = make_float2(w32[o + n * 9 + k], d->n_frames == 2 ? w32[o + (n + 6) * 9 + k] : 0.f);
      }
  }
  const int brdf_in = d->use_frames ? 8 + 6 * d->n_frames : 14;
  mp.brdf_in = brdf_in;
  if (d->brdf.n_layers > 0) {
    if ((rc = view_net(d->brdf, "brdf decoder", bv)) != NM_OK) { delete m; return rc; }
    if (bv.fi[0] != brdf_in) {
      delete m;
      return fail(NM_ERR_INVALID, "expected input width " + std::to_string(brdf_in) +
                                      ", got " + std::to_string(bv.fi[0]));
    }
    const int brdf_out = d->albedo_head ? 6 : 3;
    if (bv.fo.back() != brdf_out) {
      delete m;
      return fail(NM_ERR_INVALID, "brdf decoder output width mismatch");
    }
    if (d->use_frames && d->frame.n_layers <= 0) {
      delete m;
      return fail(NM_ERR_INVALID, "use_frames requires a frame layer");
    }
    mp.has_brdf = 1;
    mp.brdf_first = nl;
    mp.brdf_count = bv.n_layers;
    if ((rc = pack_chain(bv, pk, mp, nl, "brdf decoder")) != NM_OK) { delete m; return rc; }
    append_w32(bv, mp.precise, w32, mp, mp.brdf_first);
  }
  if (d->sampler.n_layers > 0) {
    if ((rc = view_net(d->sampler, "sampler decoder", sv)) != NM_OK) { delete m; return rc; }
    if (sv.fi[0] != 11 || sv.fo.back() != (d->sampler_isotropic ? 2 : 9)) {
      delete m;
      return fail(NM_ERR_INVALID, "sampler decoder shape mismatch");
    }
    mp.has_sampler = 1;
    mp.samp_first = nl;
    mp.samp_count = sv.n_layers;
    if ((rc = pack_chain(sv, pk, mp, nl, "sampler decoder")) != NM_OK) { delete m; return rc; }
    append_w32(sv, mp.precise, w32, mp, mp.samp_first);
  }
  for (int l = mp.brdf_first; l < mp.brdf_first + mp.brdf_count; ++l)
    m->brdf_width = m->brdf_width > mp.layers[l].n_pad ? m->brdf_width : mp.layers[l].n_pad;
  for (int l = mp.samp_first; l < mp.samp_first + mp.samp_count; ++l)
    m->sampler_width = m->sampler_width > mp.layers[l].n_pad ? m->sampler_width : mp.layers[l].n_pad;
  if (mp.dmax < 16) mp.dmax = 16;
  if (mp.dmax == 48) mp.dmax = 64;  // TMEM regions are powers of two
  mp.fast_arch = mp.precise ? -1 : detect_fast_arch(mp, bv, sv, d);
  if (mp.fast_arch >= 0) fill_fast_layers(mp, pk, fv, bv);
  mp.wblob_bytes = (uint32_t)(pk.blob.size() * 2);
  if (mp.wblob_bytes > 200 * 1024) {
    delete m;
    return fail(NM_ERR_UNSUPPORTED, "weights exceed shared memory");
  }

  // --- device upload ---------------------------------------------------------------
  DeviceGuard guard(device);
  cudaError_t e;
  const size_t lat_bytes = (size_t)m->texels * texel_bytes;
  if ((e = cudaMalloc(&m->latent, lat_bytes)) != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cudaMalloc(latent)");
  }
  e = cudaMemcpy(m->latent, d->latent, lat_bytes,
                 d->latent_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(m->latent);
    delete m;
    return cuda_fail(e, "upload latent");
  }
  if (mp.wblob_bytes == 0) pk.append(16, 1), mp.wblob_bytes = (uint32_t)(pk.blob.size() * 2);
  if ((e = cudaMalloc(&m->wblob, mp.wblob_bytes)) != cudaSuccess ||
      (e = cudaMemcpy(m->wblob, pk.blob.data(), mp.wblob_bytes, cudaMemcpyHostToDevice)) !=
          cudaSuccess) {
    cudaFree(m->latent);
    if (m->wblob) cudaFree(m->wblob);
    delete m;
    return cuda_fail(e, "upload weights");
  }
  if (w32.empty()) w32.push_back(0.f);
  if ((e = cudaMalloc(&m->w32, w32.size() * sizeof(float))) != cudaSuccess ||
      (e = cudaMemcpy(m->w32, w32.data(), w32.size() * sizeof(float), cudaMemcpyHostToDevice)) !=
          cudaSuccess) {
    cudaFree(m->latent);
    cudaFree(m->wblob);
    if (m->w32) cudaFree(m->w32);
    delete m;
    return cuda_fail(e, "upload fp32 weights");
  }
  mp.latent = reinterpret_cast<const uint4*>(m->latent);
  mp.wblob = reinterpret_cast<const uint4*>(m->wblob);
  mp.w32 = reinterpret_cast<const float*>(m->w32);
  *out = m;
  return NM_OK;
}

int nm_material_destroy(nm_material* m) {
  if (!m) return NM_OK;
  DeviceGuard guard(m->device);
  div_forget(m);
  if (m->latent) cudaFree(m->latent);
  if (m->wblob) cudaFree(m->wblob);
  if (m->w32) cudaFree(m->w32);
  delete m;
  return NM_OK;
}

int nm_material_info_get(const nm_material* m, nm_material_info* info) {
  if (!m || !info) return fail(NM_ERR_INVALID, "null argument");
  info->device = m->device;
  info->n_levels = m->mp.n_levels;
  info->latent_texels = m->texels;
  info->latent_bytes = m->texels * (m->mp.texel_fp32 ? 32 : 16);
  info->weight_bytes = (int32_t)m->mp.wblob_bytes;
  info->brdf_width = m->brdf_width;
  info->sampler_width = m->sampler_width;
  return NM_OK;
}

int nm_material_levels(const nm_material* m, int32_t* w, int32_t* h, int64_t* offset) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  for (int i = 0; i < m->mp.n_levels; ++i) {
    if (w) w[i] = m->mp.lv[i].w;
    if (h) h[i] = m->mp.lv[i].h;
    if (offset) offset[i] = m->mp.lv[i].off;
  }
  return NM_OK;
}

const void* nm_material_latent_ptr(const nm_material* m) { return m ? m->latent : nullptr; }

#define NM_CHECK_N(n)                                          \
  do {                                                         \
    if ((n) < 0) return fail(NM_ERR_INVALID, "negative batch"); \
  } while (0)

static int finish(const nm_material* m, cudaError_t e, const char* what) {
  (void)m;
  if (e == cudaErrorNotSupported)
    return fail(NM_ERR_UNSUPPORTED, std::string(what) + ": shape outside what the kernels implement");
  if (e != cudaSuccess) return cuda_fail(e, what);
  return NM_OK;
}

int nm_fetch(const nm_material* m, int64_t n, const float* uv, const float* lod,
             int32_t lod_stride, const float* u_rr, float* z_out, int32_t* level_out,
             int32_t* taps_out, float* wts_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.z_out = z_out; a.level = level_out; a.taps = taps_out; a.wts = wts_out;
  DeviceGuard guard(m->device);
  return finish(m, launch_fetch(m->mp, a, (cudaStream_t)stream), "nm_fetch");
}

int nm_fetch_trilinear(const nm_material* m, int64_t n, const float* uv, const float* lod,
                       int32_t lod_stride, float* z_out, int32_t* level_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !z_out) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = lod;  // unused
  a.z_out = z_out; a.level = level_out; a.trilinear = 1;
  DeviceGuard guard(m->device);
  return finish(m, launch_fetch(m->mp, a, (cudaStream_t)stream), "nm_fetch_trilinear");
}

int nm_fetch_f64(const nm_material* m, int64_t n, const double* uv, const double* lod, int32_t lod_stride,
                 const double* u_rr, float* z_out, int32_t* level_out, int32_t* taps_out, float* wts_out,
                 void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv64 = uv; a.lod64 = lod; a.lod_stride = lod_stride ? 1 : 0; a.urr64 = u_rr;
  a.z_out = z_out; a.level = level_out; a.taps = taps_out; a.wts = wts_out;
  DeviceGuard guard(m->device);
  return finish(m, launch_fetch(m->mp, a, (cudaStream_t)stream), "nm_fetch_f64");
}

int nm_query_f64(const nm_material* m, int32_t mode, int64_t n, const double* uv, const double* lod,
                 int32_t lod_stride, const double* u_rr, const double* wi, const double* wo, const float* u3,
                 float* rgb_out, float* albedo_out, float* ws_out, float* pdf_out, float* params9_out,
                 int32_t* level_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  const bool brdf = mode == NM_QUERY_EVAL || mode == NM_QUERY_FULL;
  const bool samp = mode == NM_QUERY_SAMPLE_PDF || mode == NM_QUERY_FULL;
  if (!brdf && !samp) return fail(NM_ERR_INVALID, "unknown query mode");
  if (!uv || !lod || !u_rr || !wi || (brdf && (!wo || !rgb_out)) || (samp && (!u3 || !ws_out || !pdf_out)))
    return fail(NM_ERR_INVALID, "null input");
  if (brdf && !m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  if (samp && !m->mp.has_sampler) return fail(NM_ERR_INVALID, "material has no sampler decoder");
  QueryArgs a{};
  a.n = n; a.uv64 = uv; a.lod64 = lod; a.lod_stride = lod_stride ? 1 : 0; a.urr64 = u_rr;
  a.wi64 = wi; a.wo64 = brdf ? wo : nullptr; a.u3 = u3; a.rgb = rgb_out; a.albedo = albedo_out; a.ws = ws_out;
  a.pdf = pdf_out; a.params9 = params9_out; a.level = level_out;
  DeviceGuard guard(m->device);
  const int kmode = mode == NM_QUERY_EVAL ? kModeEval : (mode == NM_QUERY_SAMPLE_PDF ? kModeSamplePdf : kModeQuery);
  return finish(m, launch_fused(m->mp, kmode, a, (cudaStream_t)stream), "nm_query_f64");
}

int nm_eval_spp(const nm_material* m, int64_t n, const float* uv, const float* lod, int32_t lod_stride,
                const float* u_rr, const float* wi, const float* wo, int32_t spp, float* img_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (spp <= 0 || (spp & (spp - 1))) return fail(NM_ERR_INVALID, "spp must be a power of two");
  if (n % spp) return fail(NM_ERR_INVALID, "the batch must be whole pixels (n a multiple of spp)");
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !wo || !img_out) return fail(NM_ERR_INVALID, "null input");
  if (!m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  int lg = 0;
  while ((1 << lg) < spp) ++lg;
  DeviceGuard guard(m->device);
  cudaError_t e = cudaMemsetAsync(img_out, 0, (size_t)(n / spp) * 12, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "nm_eval_spp");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.wo = wo; a.img = img_out; a.spp_log2 = lg;
  return finish(m, launch_fused(m->mp, kModeEval, a, (cudaStream_t)stream), "nm_eval_spp");
}

int nm_eval(const nm_material* m, int64_t n, const float* uv, const float* lod,
            int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
            float* rgb_out, float* albedo_out, int32_t* level_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !wo || !rgb_out) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.wo = wo; a.rgb = rgb_out; a.albedo = albedo_out; a.level = level_out;
  DeviceGuard guard(m->device);
  if (!m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  return finish(m, launch_fused(m->mp, kModeEval, a, (cudaStream_t)stream), "nm_eval");
}

int nm_eval_debug_tw(const nm_material* m, int64_t n, const float* uv, const float* lod,
                     int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
                     float* rgb_out, float* dbg_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !wo || !rgb_out || !dbg_out) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.wo = wo; a.rgb = rgb_out; a.dbg = dbg_out;
  DeviceGuard guard(m->device);
  const cudaError_t e = launch_fast(m->mp, kModeEval, a, (cudaStream_t)stream);
  if (e == cudaErrorNotSupported) return fail(NM_ERR_UNSUPPORTED, "material has no pipelined kernel");
  return finish(m, e, "nm_eval_debug_tw");
}

// Host-buffer eval.  Pinned (page-locked, UVA-mapped) buffers: zero-copy —
// ONE fused-kernel launch whose TMA input loads and rgb stores go over PCIe
// directly (measured 1.21 vs 1.07 G q/s for the staged pipeline below: no
// copy-engine per-copy gaps, no pipeline head/tail; profiles/r01_e2e_probe.txt).
// Otherwise (pageable memory): the batch streams through the GPU in chunks over a ring
// of NMQ_HOST_SLOTS device staging slots and three internal streams — one
// for all H2D copies (chunks in order: concurrent H2D copies on several copy
// engines would only share PCIe and finish together, delaying the first
// kernel), one for the fused kernels, one for the D2H copies (the opposite
// PCIe direction, overlapped with the later chunks' H2D).  Blocking: returns
// when rgb_out (host) is complete.  Device staging is per device, grow-only.
namespace {
#ifndef NMQ_HOST_SLOTS
#define NMQ_HOST_SLOTS 4  // chunks in flight: H2D can run ahead of the D2H of older chunks
#endif
struct HostStage {
  std::mutex mu;
  char* buf = nullptr;
  size_t bytes = 0;
  cudaStream_t h2d = nullptr, run = nullptr, d2h = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_in[NMQ_HOST_SLOTS] = {}, ev_k[NMQ_HOST_SLOTS] = {}, ev_out[NMQ_HOST_SLOTS] = {};
};
HostStage g_stage[16];

// ---- pageable host buffers: pinned bounce pipeline ---------------------------
// Pageable memory cannot be read by DMA; the driver's own staging copies it
// through small pinned buffers on the calling thread (~12 GB/s for the C2
// inputs).  Here a pool of host threads copies each chunk into a pinned
// slot (and the results out of one), the copy engines move pinned slots at
// PCIe speed, and the chunks pipeline over NMQ_HOST_SLOTS slots: copy-in of
// chunk i, DMA + kernel of i-1..i-3 and copy-out of i-3 overlap.  The
// reference-dtype variant widens rgb / albedo to float64 and levels to int64
// on the device (neural.py:303 returns them so), so the host never converts.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // never destroyed: workers idle at exit
    return *p;
  }
  // f(i) for i in [0, tasks), on the pool and the calling thread; returns when done
  void run(int tasks, const std::function<void(int)>& f) {
    if (tasks <= 0) return;
    if (workers_.empty() || tasks == 1) {
      for (int i = 0; i < tasks; ++i) f(i);
      return;
    }
    std::lock_guard<std::mutex> serial(run_mu_);
    {
      std::lock_guard<std::mutex> l(mu_);
      job_ = &f;
      ntask_ = tasks;
      next_.store(0);
      pending_ = (int)workers_.size() + 1;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> l(mu_);
    done_cv_.wait(l, [&] { return pending_ == 0; });
  }

 private:
  HostPool() {
    // 8 by default (measured on the 16-core B200 hosts: 8 > 6 > 12 > 16 for
    // the C2 drop-in call — more threads contend with the driver's own)
    int n = (int)std::thread::hardware_concurrency();
    n = n > 8 ? 8 : n;
    if (const char* v = getenv("NMQ_HOST_THREADS")) n = atoi(v);
    n = n < 1 ? 1 : (n > 32 ? 32 : n);
    for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [&] { return gen_ != seen; });
        seen = gen_;
      }
      work();
    }
  }
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= ntask_) break;
      (*job_)(i);
    }
    std::lock_guard<std::mutex> l(mu_);
    if (--pending_ == 0) done_cv_.notify_all();
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  int ntask_ = 0, pending_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
};

struct CopyJob {
  void* dst;
  const void* src;
  size_t bytes;
};
// memcpy a list of (possibly large) ranges on the pool in ~1 MiB pieces
void parallel_copy(const std::vector<CopyJob>& jobs) {
  constexpr size_t kPiece = size_t(1) << 20;
  std::vector<CopyJob> pieces;
  for (const CopyJob& j : jobs)
    for (size_t o = 0; o < j.bytes; o += kPiece)
      pieces.push_back({(char*)j.dst + o, (const char*)j.src + o, j.bytes - o < kPiece ? j.bytes - o : kPiece});
  HostPool::get().run((int)pieces.size(), [&](int i) { memcpy(pieces[i].dst, pieces[i].src, pieces[i].bytes); });
}

__global__ void widen_kernel(int64_t c, const float* __restrict__ rgb, const float* __restrict__ alb,
                             const int32_t* __restrict__ lv, double* __restrict__ rgb64,
                             double* __restrict__ alb64, int64_t* __restrict__ lv64) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * c; i += stride) {
    rgb64[i] = rgb[i];
    if (alb) alb64[i] = alb[i];
    if (lv && i < c) lv64[i] = lv[i];
  }
}

struct HostIo {
  const float *uv, *lod;
  int32_t lod_stride;
  const float *u_rr, *wi, *wo;
  void *rgb, *albedo, *level;  // float / int32, or double / int64 when wide
  bool wide;
};

struct BounceStage {
  std::mutex mu;
  char* pin = nullptr;  // pinned: per slot inputs (40 B/row) | outputs (56 B/row)
  char* dev = nullptr;  // device: per slot inputs | fp32 outputs (28 B/row) | wide outputs (56 B/row)
  int64_t chunk = 0;
  cudaStream_t h2d = nullptr, run = nullptr, d2h = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_in[NMQ_HOST_SLOTS] = {}, ev_k[NMQ_HOST_SLOTS] = {}, ev_out[NMQ_HOST_SLOTS] = {};
};
BounceStage g_bounce[16];
constexpr size_t kInRow = 8 + 4 + 4 + 12 + 12, kOutRow = 24 + 24 + 8, kDevOutRow = 12 + 12 + 4;

bool is_pinned(const void* p) {
  if (!p) return true;  // absent optional buffer
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int host_eval_bounce(const nm_material* m, int64_t n, const HostIo& io, int64_t chunk, void* stream) {
  BounceStage& B = g_bounce[m->device & 15];
  std::lock_guard<std::mutex> lock(B.mu);
  cudaError_t e;
  if (B.chunk < chunk) {
    if (B.pin) cudaFreeHost(B.pin);
    if (B.dev) cudaFree(B.dev);
    B.pin = B.dev = nullptr;
    B.chunk = 0;
    if ((e = cudaHostAlloc((void**)&B.pin, NMQ_HOST_SLOTS * (size_t)chunk * (kInRow + kOutRow), 0)) != cudaSuccess)
      return cuda_fail(e, "host-eval pinned staging");
    if ((e = cudaMalloc(&B.dev, NMQ_HOST_SLOTS * (size_t)chunk * (kInRow + kDevOutRow + kOutRow))) != cudaSuccess)
      return cuda_fail(e, "host-eval device staging");
    B.chunk = chunk;
  }
  if (!B.h2d) {
    for (cudaStream_t* st : {&B.h2d, &B.run, &B.d2h}) cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&B.ev_start, cudaEventDisableTiming);
    for (int i = 0; i < NMQ_HOST_SLOTS; ++i) {
      cudaEventCreateWithFlags(&B.ev_in[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&B.ev_k[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&B.ev_out[i], cudaEventDisableTiming);
    }
  }
  const int64_t ck = B.chunk;
  cudaEventRecord(B.ev_start, (cudaStream_t)stream);  // after prior work on the caller's stream
  for (cudaStream_t st : {B.h2d, B.run, B.d2h}) cudaStreamWaitEvent(st, B.ev_start, 0);
  const size_t ob = io.wide ? 8 : 4;  // output element bytes
  struct Slot {
    char *pin_in, *pin_out, *dev_in, *dev_out, *dev_wide;
  };
  auto slot = [&](int s) {
    Slot q;
    q.pin_in = B.pin + (size_t)s * ck * kInRow;
    q.pin_out = B.pin + (size_t)NMQ_HOST_SLOTS * ck * kInRow + (size_t)s * ck * kOutRow;
    q.dev_in = B.dev + (size_t)s * ck * kInRow;
    q.dev_out = B.dev + (size_t)NMQ_HOST_SLOTS * ck * kInRow + (size_t)s * ck * kDevOutRow;
    q.dev_wide = B.dev + (size_t)NMQ_HOST_SLOTS * ck * (kInRow + kDevOutRow) + (size_t)s * ck * kOutRow;
    return q;
  };
  const int64_t nch = (n + ck - 1) / ck;
  // page-locked result buffers take the DMA directly (no pinned slot, no host copy)
  const bool direct_out = is_pinned(io.rgb) && is_pinned(io.albedo) && is_pinned(io.level);
  auto drain = [&](int64_t cj) -> int {  // results of chunk cj -> the caller's buffers
    const int s = (int)(cj % NMQ_HOST_SLOTS);
    const int64_t c0 = cj * ck, c = n - c0 < ck ? n - c0 : ck;
    cudaError_t err = cudaEventSynchronize(B.ev_out[s]);
    if (err != cudaSuccess) return cuda_fail(err, "nm_eval_host");
    if (direct_out) return NM_OK;
    const Slot q = slot(s);
    std::vector<CopyJob> jobs{{(char*)io.rgb + 3 * c0 * ob, q.pin_out, (size_t)c * 3 * ob}};
    if (io.albedo) jobs.push_back({(char*)io.albedo + 3 * c0 * ob, q.pin_out + (size_t)ck * 3 * ob, (size_t)c * 3 * ob});
    if (io.level) jobs.push_back({(char*)io.level + c0 * ob, q.pin_out + (size_t)ck * 6 * ob, (size_t)c * ob});
    parallel_copy(jobs);
    return NM_OK;
  };
  for (int64_t ci = 0; ci < nch; ++ci) {
    const int s = (int)(ci % NMQ_HOST_SLOTS);
    const bool reuse = ci >= NMQ_HOST_SLOTS;
    const int64_t c0 = ci * ck, c = n - c0 < ck ? n - c0 : ck;
    const Slot q = slot(s);
    // inputs: pageable -> pinned slot (host threads) -> device slot (DMA)
    if (reuse && (e = cudaEventSynchronize(B.ev_in[s])) != cudaSuccess) return cuda_fail(e, "nm_eval_host");
    float* p_uv = (float*)q.pin_in;
    float* p_lod = p_uv + 2 * ck;
    float* p_urr = p_lod + ck;
    float* p_wi = p_urr + ck;
    float* p_wo = p_wi + 3 * ck;
    parallel_copy({{p_uv, io.uv + 2 * c0, (size_t)c * 8},
                   {p_lod, io.lod_stride ? io.lod + c0 : io.lod, io.lod_stride ? (size_t)c * 4 : 4},
                   {p_urr, io.u_rr + c0, (size_t)c * 4},
                   {p_wi, io.wi + 3 * c0, (size_t)c * 12},
                   {p_wo, io.wo + 3 * c0, (size_t)c * 12}});
    if (reuse) cudaStreamWaitEvent(B.h2d, B.ev_k[s], 0);  // the older chunk's kernel has read the slot
    cudaMemcpyAsync(q.dev_in, q.pin_in, (size_t)ck * kInRow, cudaMemcpyHostToDevice, B.h2d);
    cudaEventRecord(B.ev_in[s], B.h2d);
    // kernel (+ widening) on the run stream
    cudaStreamWaitEvent(B.run, B.ev_in[s], 0);
    if (reuse) cudaStreamWaitEvent(B.run, B.ev_out[s], 0);  // the older chunk's results have left
    float* d_uv = (float*)q.dev_in;
    float* d_rgb = (float*)q.dev_out;
    float* d_alb = d_rgb + 3 * ck;
    int32_t* d_lv = (int32_t*)(d_alb + 3 * ck);
    QueryArgs a{};
    a.n = c; a.uv = d_uv; a.lod = d_uv + 2 * ck; a.lod_stride = io.lod_stride ? 1 : 0; a.u_rr = d_uv + 3 * ck;
    a.wi = d_uv + 4 * ck; a.wo = d_uv + 7 * ck; a.rgb = d_rgb;
    a.albedo = io.albedo ? d_alb : nullptr;
    a.level = io.level ? d_lv : nullptr;
    if ((e = launch_fused(m->mp, kModeEval, a, B.run)) != cudaSuccess) return cuda_fail(e, "nm_eval_host");
    const char* out_src = q.dev_out;
    if (io.wide) {
      double* w = (double*)q.dev_wide;
      widen_kernel<<<148 * 4, 256, 0, B.run>>>(c, d_rgb, a.albedo, a.level, w, w + 3 * ck, (int64_t*)(w + 6 * ck));
      ++g_launches;
      out_src = q.dev_wide;
    }
    cudaEventRecord(B.ev_k[s], B.run);
    // results -> pinned slot (DMA; same layout as the device slot: rgb | albedo
    // | level), or straight into page-locked result buffers
    cudaStreamWaitEvent(B.d2h, B.ev_k[s], 0);
    char* o_rgb = direct_out ? (char*)io.rgb + 3 * c0 * ob : q.pin_out;
    char* o_alb = direct_out ? (char*)io.albedo + 3 * c0 * ob : q.pin_out + (size_t)ck * 3 * ob;
    char* o_lv = direct_out ? (char*)io.level + c0 * ob : q.pin_out + (size_t)ck * 6 * ob;
    cudaMemcpyAsync(o_rgb, out_src, (size_t)c * 3 * ob, cudaMemcpyDeviceToHost, B.d2h);
    if (io.albedo)
      cudaMemcpyAsync(o_alb, out_src + (size_t)ck * 3 * ob, (size_t)c * 3 * ob, cudaMemcpyDeviceToHost, B.d2h);
    if (io.level)
      cudaMemcpyAsync(o_lv, out_src + (size_t)ck * 6 * ob, (size_t)c * ob, cudaMemcpyDeviceToHost, B.d2h);
    cudaEventRecord(B.ev_out[s], B.d2h);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "nm_eval_host");
    if (ci >= NMQ_HOST_SLOTS - 1) {
      const int rc = drain(ci - (NMQ_HOST_SLOTS - 1));
      if (rc != NM_OK) return rc;
    }
  }
  for (int64_t cj = nch > NMQ_HOST_SLOTS - 1 ? nch - (NMQ_HOST_SLOTS - 1) : 0; cj < nch; ++cj) {
    const int rc = drain(cj);
    if (rc != NM_OK) return rc;
  }
  return NM_OK;
}
}  // namespace

int nm_eval_host(const nm_material* m, int64_t n, const float* uv, const float* lod,
                 int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
                 float* rgb_out, float* albedo_out, int32_t* level_out, int64_t chunk, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !wo || !rgb_out) return fail(NM_ERR_INVALID, "null input");
  if (!m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  if (chunk <= 0) chunk = (int64_t)1 << 19;
  chunk = (chunk + 127) / 128 * 128;
  DeviceGuard guard(m->device);
  cudaError_t e;
  {
    // zero-copy: when every buffer is pinned (page-locked, mapped under UVA),
    // the fused kernel reads the inputs and writes rgb over PCIe directly —
    // no staging copies, no chunk pipeline head/tail
    static const int zc = [] {  // NMQ_HOST_ZEROCOPY=0: always stage (A/B)
      const char* v = getenv("NMQ_HOST_ZEROCOPY");
      return v ? atoi(v) : 1;
    }();
    const void* hp[8] = {uv, lod, u_rr, wi, wo, rgb_out, albedo_out, level_out};
    void* dp[8] = {};
    bool mapped = zc != 0;
    for (int i = 0; i < 8 && mapped; ++i) {
      if (!hp[i]) continue;  // optional outputs
      cudaPointerAttributes at;
      if (cudaPointerGetAttributes(&at, hp[i]) != cudaSuccess || at.type != cudaMemoryTypeHost ||
          !at.devicePointer) {
        cudaGetLastError();
        mapped = false;
      } else {
        dp[i] = at.devicePointer;
      }
    }
    if (mapped) {
      QueryArgs a{};
      a.n = n; a.uv = (const float*)dp[0]; a.lod = (const float*)dp[1]; a.lod_stride = lod_stride ? 1 : 0;
      a.u_rr = (const float*)dp[2]; a.wi = (const float*)dp[3]; a.wo = (const float*)dp[4];
      a.rgb = (float*)dp[5]; a.albedo = (float*)dp[6]; a.level = (int32_t*)dp[7];
      if ((e = launch_fused(m->mp, kModeEval, a, (cudaStream_t)stream)) != cudaSuccess)
        return cuda_fail(e, "nm_eval_host");
      if ((e = cudaStreamSynchronize((cudaStream_t)stream)) != cudaSuccess) return cuda_fail(e, "nm_eval_host");
      return NM_OK;
    }
  }
  {
    static const int bounce = [] {  // NMQ_HOST_BOUNCE=0: driver-staged pageable copies (A/B)
      const char* v = getenv("NMQ_HOST_BOUNCE");
      return v ? atoi(v) : 1;
    }();
    if (bounce) {
      const HostIo io{uv, lod, lod_stride, u_rr, wi, wo, rgb_out, albedo_out, level_out, false};
      return host_eval_bounce(m, n, io, chunk, stream);
    }
  }
  HostStage& H = g_stage[m->device & 15];
  std::lock_guard<std::mutex> lock(H.mu);
  const size_t per_row = 8 + 4 + 4 + 12 + 12 + 12 + 12 + 4;  // uv lod u_rr wi wo | rgb albedo level
  const size_t need = NMQ_HOST_SLOTS * (size_t)chunk * per_row + 1024;
  if (H.bytes < need) {
    if (H.buf) cudaFree(H.buf);
    H.buf = nullptr;
    H.bytes = 0;
    if ((e = cudaMalloc(&H.buf, need)) != cudaSuccess) return cuda_fail(e, "host-eval staging");
    H.bytes = need;
  }
  if (!H.h2d) {
    for (cudaStream_t* st : {&H.h2d, &H.run, &H.d2h}) cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&H.ev_start, cudaEventDisableTiming);
    for (int i = 0; i < NMQ_HOST_SLOTS; ++i) {
      cudaEventCreateWithFlags(&H.ev_in[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&H.ev_k[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&H.ev_out[i], cudaEventDisableTiming);
    }
  }
  cudaEventRecord(H.ev_start, (cudaStream_t)stream);  // after prior work on the caller's stream
  for (cudaStream_t st : {H.h2d, H.run, H.d2h}) cudaStreamWaitEvent(st, H.ev_start, 0);
  for (int64_t c0 = 0, ci = 0; c0 < n; c0 += chunk, ++ci) {
    const int64_t c = n - c0 < chunk ? n - c0 : chunk;
    const int s = (int)(ci % NMQ_HOST_SLOTS);
    const bool reuse = ci >= NMQ_HOST_SLOTS;  // slot held an older chunk
    char* base = H.buf + (size_t)s * chunk * per_row;
    float* d_uv = (float*)base;
    float* d_lod = d_uv + 2 * chunk;
    float* d_urr = d_lod + chunk;
    float* d_wi = d_urr + chunk;
    float* d_wo = d_wi + 3 * chunk;
    float* d_rgb = d_wo + 3 * chunk;
    float* d_alb = d_rgb + 3 * chunk;
    int32_t* d_lv = reinterpret_cast<int32_t*>(d_alb + 3 * chunk);
    if (reuse) cudaStreamWaitEvent(H.h2d, H.ev_k[s], 0);  // older chunk's kernel has read the inputs
    cudaMemcpyAsync(d_uv, uv + 2 * c0, c * 8, cudaMemcpyHostToDevice, H.h2d);
    if (lod_stride) cudaMemcpyAsync(d_lod, lod + c0, c * 4, cudaMemcpyHostToDevice, H.h2d);
    else cudaMemcpyAsync(d_lod, lod, 4, cudaMemcpyHostToDevice, H.h2d);
    cudaMemcpyAsync(d_urr, u_rr + c0, c * 4, cudaMemcpyHostToDevice, H.h2d);
    cudaMemcpyAsync(d_wi, wi + 3 * c0, c * 12, cudaMemcpyHostToDevice, H.h2d);
    cudaMemcpyAsync(d_wo, wo + 3 * c0, c * 12, cudaMemcpyHostToDevice, H.h2d);
    cudaEventRecord(H.ev_in[s], H.h2d);
    cudaStreamWaitEvent(H.run, H.ev_in[s], 0);
    if (reuse) cudaStreamWaitEvent(H.run, H.ev_out[s], 0);  // older chunk's rgb has left
    QueryArgs a{};
    a.n = c; a.uv = d_uv; a.lod = d_lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = d_urr;
    a.wi = d_wi; a.wo = d_wo; a.rgb = d_rgb;
    a.albedo = albedo_out ? d_alb : nullptr;
    a.level = level_out ? d_lv : nullptr;
    if ((e = launch_fused(m->mp, kModeEval, a, H.run)) != cudaSuccess) return cuda_fail(e, "nm_eval_host");
    cudaEventRecord(H.ev_k[s], H.run);
    cudaStreamWaitEvent(H.d2h, H.ev_k[s], 0);
    cudaMemcpyAsync(rgb_out + 3 * c0, d_rgb, c * 12, cudaMemcpyDeviceToHost, H.d2h);
    if (albedo_out) cudaMemcpyAsync(albedo_out + 3 * c0, d_alb, c * 12, cudaMemcpyDeviceToHost, H.d2h);
    if (level_out) cudaMemcpyAsync(level_out + c0, d_lv, c * 4, cudaMemcpyDeviceToHost, H.d2h);
    cudaEventRecord(H.ev_out[s], H.d2h);
  }
  for (cudaStream_t st : {H.h2d, H.run, H.d2h})
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "nm_eval_host");
  return NM_OK;
}

int nm_eval_host_ref(const nm_material* m, int64_t n, const float* uv, const float* lod, int32_t lod_stride,
                     const float* u_rr, const float* wi, const float* wo, double* rgb_out, double* albedo_out,
                     int64_t* level_out, int64_t chunk, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !wo || !rgb_out) return fail(NM_ERR_INVALID, "null input");
  if (!m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  if (chunk <= 0) chunk = (int64_t)1 << 18;
  chunk = (chunk + 127) / 128 * 128;
  DeviceGuard guard(m->device);
  const HostIo io{uv, lod, lod_stride, u_rr, wi, wo, rgb_out, albedo_out, level_out, true};
  return host_eval_bounce(m, n, io, chunk, stream);
}

int nm_eval_z(const nm_material* m, int64_t n, const float* z, const float* wi, const float* wo,
              float* rgb_out, float* albedo_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!z || !wi || !wo || !rgb_out) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.z = z; a.wi = wi; a.wo = wo; a.rgb = rgb_out; a.albedo = albedo_out;
  DeviceGuard guard(m->device);
  if (!m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  return finish(m, launch_fused(m->mp, kModeEvalZ, a, (cudaStream_t)stream), "nm_eval_z");
}

int nm_eval_z_f64(const nm_material* m, int64_t n, const float* z, const double* wi, const double* wo,
                  float* rgb_out, float* albedo_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!z || !wi || !wo || !rgb_out) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.z = z; a.wi64 = wi; a.wo64 = wo; a.rgb = rgb_out; a.albedo = albedo_out;
  DeviceGuard guard(m->device);
  if (!m->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
  return finish(m, launch_fused(m->mp, kModeEvalZ, a, (cudaStream_t)stream), "nm_eval_z_f64");
}

int nm_decoder_inputs(const nm_material* m, int64_t n, const float* z, const float* wi, const float* wo,
                      const double* wi64, const double* wo64, uint16_t* x16_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!z || !x16_out || !((wi && wo) || (wi64 && wo64))) return fail(NM_ERR_INVALID, "null input");
  if (!m->mp.use_frames || m->mp.precise) return fail(NM_ERR_INVALID, "needs an fp16 material with learned frames");
  DeviceGuard guard(m->device);
  return finish(m, launch_decoder_inputs(m->mp, n, z, wi64 ? nullptr : wi, wo, wi64, wo64, (uint32_t*)x16_out,
                                         (cudaStream_t)stream), "nm_decoder_inputs");
}

int nm_infer_proxy(const nm_material* m, int64_t n, const float* z, const float* wi,
                   float* params9_out, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!z || !wi || !params9_out) return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.z = z; a.wi = wi; a.params9 = params9_out;
  DeviceGuard guard(m->device);
  if (!m->mp.has_sampler) return fail(NM_ERR_INVALID, "material has no sampler decoder");
  return finish(m, launch_fused(m->mp, kModeProxyZ, a, (cudaStream_t)stream), "nm_infer_proxy");
}

int nm_sample(int64_t n, const float* params9, const float* wi, const float* u3, float* wo_out,
              void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!params9 || !wi || !u3 || !wo_out) return fail(NM_ERR_INVALID, "null input");
  return finish(nullptr, launch_sample(n, params9, wi, u3, wo_out, (cudaStream_t)stream),
                "nm_sample");
}

int nm_pdf(int64_t n, const float* params9, const float* wi, const float* wo, float* pdf_out,
           void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!params9 || !wi || !wo || !pdf_out) return fail(NM_ERR_INVALID, "null input");
  return finish(nullptr, launch_pdf(n, params9, wi, wo, pdf_out, (cudaStream_t)stream), "nm_pdf");
}

int nm_sample_pdf(const nm_material* m, int64_t n, const float* uv, const float* lod,
                  int32_t lod_stride, const float* u_rr, const float* wi, const float* u3,
                  float* ws_out, float* pdf_out, float* params9_out, int32_t* level_out,
                  void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !u3 || !ws_out || !pdf_out)
    return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.u3 = u3; a.ws = ws_out; a.pdf = pdf_out; a.params9 = params9_out;
  a.level = level_out;
  DeviceGuard guard(m->device);
  if (!m->mp.has_sampler) return fail(NM_ERR_INVALID, "material has no sampler decoder");
  return finish(m, launch_fused(m->mp, kModeSamplePdf, a, (cudaStream_t)stream), "nm_sample_pdf");
}

int nm_query(const nm_material* m, int64_t n, const float* uv, const float* lod,
             int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
             const float* u3, float* rgb_out, float* ws_out, float* pdf_out, int32_t* level_out,
             void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !lod || !u_rr || !wi || !wo || !u3 || !rgb_out || !ws_out || !pdf_out)
    return fail(NM_ERR_INVALID, "null input");
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.wo = wo; a.u3 = u3; a.rgb = rgb_out; a.ws = ws_out; a.pdf = pdf_out;
  a.level = level_out;
  DeviceGuard guard(m->device);
  if (!m->mp.has_brdf || !m->mp.has_sampler)
    return fail(NM_ERR_INVALID, "material needs both decoders");
  return finish(m, launch_fused(m->mp, kModeQuery, a, (cudaStream_t)stream), "nm_query");
}

int nm_texel_grads(const nm_material* m, int64_t n, const float* uv, const int32_t* level,
                   const float* z_grad, float* grad_texels, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null material");
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!uv || !level || !z_grad || !grad_texels) return fail(NM_ERR_INVALID, "null input");
  DeviceGuard guard(m->device);
  return finish(m, launch_texel_grads(m->mp, n, uv, level, z_grad, grad_texels, (cudaStream_t)stream),
                "nm_texel_grads");
}

int nm_mlp_create(const nm_net_desc* net, int device, nm_mlp** out) {
  if (!net || !out) return fail(NM_ERR_INVALID, "null argument");
  *out = nullptr;
  NetView v;
  int rc;
  nm_net_desc d = *net;
  if (!d.packed) {  // fp32-only description: view_net wants a packed pointer
    static const uint16_t dummy = 0;
    d.packed = &dummy;
  }
  if ((rc = view_net(d, "network", v)) != NM_OK) return rc;
  if (!net->weights) return fail(NM_ERR_INVALID, "fp32 weights required");
  if (v.n_layers > kMaxLayers) return fail(NM_ERR_UNSUPPORTED, "too many layers");
  nm_mlp* m = new nm_mlp();
  m->device = device;
  m->n_layers = v.n_layers;
  int32_t floats = 0;
  for (int l = 0; l < v.n_layers; ++l) {
    if (v.fi[l] > 64 || v.fo[l] > 64) {
      delete m;
      return fail(NM_ERR_UNSUPPORTED, "training kernels handle layers up to 64 wide");
    }
    m->fi[l] = v.fi[l];
    m->fo[l] = v.fo[l];
    m->act[l] = v.act[l];
    floats += v.fo[l] * (v.fi[l] + 1);
  }
  m->w_floats = floats;
  DeviceGuard guard(device);
  cudaError_t e;
  if ((e = cudaMalloc(&m->w, (size_t)floats * 4)) != cudaSuccess) {
    delete m;
    return cuda_fail(e, "cudaMalloc(mlp weights)");
  }
  if ((e = cudaMemcpy(m->w, net->weights, (size_t)floats * 4, cudaMemcpyHostToDevice)) != cudaSuccess) {
    cudaFree(m->w);
    delete m;
    return cuda_fail(e, "upload mlp weights");
  }
  *out = m;
  return NM_OK;
}

int nm_mlp_set_weights(nm_mlp* m, const float* weights) {
  if (!m || !weights) return fail(NM_ERR_INVALID, "null argument");
  DeviceGuard guard(m->device);
  const cudaError_t e = cudaMemcpy(m->w, weights, (size_t)m->w_floats * 4, cudaMemcpyHostToDevice);
  return e == cudaSuccess ? NM_OK : cuda_fail(e, "nm_mlp_set_weights");
}

int nm_mlp_destroy(nm_mlp* m) {
  if (!m) return NM_OK;
  DeviceGuard guard(m->device);
  cudaFree(m->w);
  delete m;
  return NM_OK;
}

int32_t nm_mlp_params(const nm_mlp* m) { return m ? m->w_floats : 0; }

static size_t mlp_cache_layout(const nm_mlp* m, int64_t B, size_t* pre_off, size_t* g_off) {
  size_t widths = 0;
  for (int l = 0; l < m->n_layers; ++l) widths += (size_t)m->fo[l];
  const size_t x_bytes = ((size_t)m->fi[0] * B * 4 + 255) & ~(size_t)255;
  const size_t pre_bytes = (widths * B * 4 + 255) & ~(size_t)255;
  *pre_off = x_bytes;
  *g_off = x_bytes + pre_bytes;
  return x_bytes + pre_bytes + widths * B * 8;
}

size_t nm_mlp_cache_bytes(const nm_mlp* m, int64_t batch) {
  if (!m || batch < 0) return 0;
  size_t a, b;
  return mlp_cache_layout(m, batch, &a, &b);
}

int nm_mlp_forward_cached(const nm_mlp* m, int64_t batch, const float* x, float* out, void* cache,
                          void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null network");
  NM_CHECK_N(batch);
  if (batch == 0) return NM_OK;
  if (!x || !out || !cache) return fail(NM_ERR_INVALID, "null input");
  size_t pre_off, g_off;
  mlp_cache_layout(m, batch, &pre_off, &g_off);
  char* c = (char*)cache;
  DeviceGuard guard(m->device);
  return finish(nullptr,
                launch_mlp_forward(m->fi, m->fo, m->act, m->n_layers, m->w, m->w_floats, batch, x,
                                   (float*)c, (float*)(c + pre_off), out, (cudaStream_t)stream),
                "nm_mlp_forward_cached");
}

int nm_mlp_backward(const nm_mlp* m, int64_t batch, void* cache, const float* out_grad,
                    double* dparams, double* dx, void* stream) {
  if (!m) return fail(NM_ERR_INVALID, "null network");
  NM_CHECK_N(batch);
  if (!cache || !out_grad || !dparams || !dx) return fail(NM_ERR_INVALID, "null input");
  size_t pre_off, g_off;
  mlp_cache_layout(m, batch, &pre_off, &g_off);
  char* c = (char*)cache;
  DeviceGuard guard(m->device);
  if (batch == 0) {
    const cudaError_t e = cudaMemsetAsync(dparams, 0, (size_t)m->w_floats * 8, (cudaStream_t)stream);
    return e == cudaSuccess ? NM_OK : cuda_fail(e, "nm_mlp_backward");
  }
  return finish(nullptr,
                launch_mlp_backward(m->fi, m->fo, m->act, m->n_layers, m->w, m->w_floats, batch,
                                    (const float*)c, (const float*)(c + pre_off), out_grad,
                                    (double*)(c + g_off), dparams, dx, (cudaStream_t)stream),
                "nm_mlp_backward");
}

int nm_kl_sample(int64_t b, int32_t use_frames, int32_t n_frames, int32_t isotropic, const float* raw_s,
                 const float* raw_f, const float* z, const double* wi, const double* u_d,
                 const double* u_s, float* x2_out, double* scratch, void* stream) {
  NM_CHECK_N(b);
  if (b == 0) return NM_OK;
  if (!raw_s || !z || !wi || !u_d || !u_s || !x2_out || !scratch || (use_frames && !raw_f))
    return fail(NM_ERR_INVALID, "null input");
  if (use_frames && (n_frames < 1 || n_frames > 4)) return fail(NM_ERR_UNSUPPORTED, "1..4 frames");
  return finish(nullptr, launch_kl_sample(b, use_frames != 0, n_frames, isotropic != 0, raw_s, raw_f, z,
                                          wi, u_d, u_s, x2_out, scratch, (cudaStream_t)stream),
                "nm_kl_sample");
}

int nm_kl_target(int64_t b, int32_t out_w, const float* y, const double* scratch, double* target_out,
                 double* lum_out, float* out_grad, void* stream) {
  NM_CHECK_N(b);
  if (b == 0) return NM_OK;
  if (!y || !scratch || !target_out || !lum_out || !out_grad) return fail(NM_ERR_INVALID, "null input");
  if (out_w < 3) return fail(NM_ERR_INVALID, "decoder output narrower than 3");
  return finish(nullptr, launch_kl_target(b, out_w, y, scratch, target_out, lum_out, out_grad,
                                          (cudaStream_t)stream),
                "nm_kl_target");
}

int nm_kl_target_dir(int64_t b, int32_t use_frames, int32_t n_frames, const float* raw_f,
                     const double* dx, const double* scratch, const double* lum, double* dtarget_out,
                     void* stream) {
  NM_CHECK_N(b);
  if (b == 0) return NM_OK;
  if (!dx || !scratch || !lum || !dtarget_out || (use_frames && !raw_f))
    return fail(NM_ERR_INVALID, "null input");
  if (use_frames && (n_frames < 1 || n_frames > 4)) return fail(NM_ERR_UNSUPPORTED, "1..4 frames");
  return finish(nullptr, launch_kl_target_dir(b, use_frames != 0, n_frames, raw_f, dx, scratch, lum,
                                              dtarget_out, (cudaStream_t)stream),
                "nm_kl_target_dir");
}

int nm_kl_grad(int64_t b, int32_t isotropic, const float* raw_s, const double* wi,
               const double* scratch, const double* target, const double* dtarget, float* draw_out,
               double* loss_rows, void* stream) {
  NM_CHECK_N(b);
  if (b == 0) return NM_OK;
  if (!raw_s || !wi || !scratch || !target || !dtarget || !draw_out || !loss_rows)
    return fail(NM_ERR_INVALID, "null input");
  return finish(nullptr, launch_kl_grad(b, isotropic != 0, raw_s, wi, scratch, target, dtarget, draw_out,
                                        loss_rows, (cudaStream_t)stream),
                "nm_kl_grad");
}

int nm_footprint_level(int64_t n, const double* area_texels, int32_t n_levels, double* level_out,
                       void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!area_texels || !level_out) return fail(NM_ERR_INVALID, "null input");
  if (n_levels < 1) return fail(NM_ERR_INVALID, "n_levels must be >= 1");
  return finish(nullptr, launch_footprint_level(n, area_texels, n_levels, level_out, (cudaStream_t)stream),
                "nm_footprint_level");
}

int nm_cone_level(int64_t n, const float* cone_w, const float* cone_s, const float* t,
                  const float* cos_hit, const float* density, int32_t density_stride,
                  int32_t n_levels, float* lod_out, void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!cone_w || !cone_s || !t || !cos_hit || !density || !lod_out)
    return fail(NM_ERR_INVALID, "null input");
  if (n_levels < 1) return fail(NM_ERR_INVALID, "n_levels must be >= 1");
  return finish(nullptr, launch_cone_level(n, cone_w, cone_s, t, cos_hit, density,
                                           density_stride ? 1 : 0, n_levels, lod_out,
                                           (cudaStream_t)stream),
                "nm_cone_level");
}

size_t nm_multi_workspace_bytes(int64_t n, int32_t n_mats) {
  if (n < 0 || n_mats <= 0) return 0;
  const size_t div = (size_t)n_mats * sizeof(MatParams) + 256;
  const size_t bin = multi_workspace_bytes(n, n_mats);
  return div > bin ? div : bin;
}

static int multi_prologue(const nm_material* const* mats, int32_t n_mats, int64_t n, bool need_brdf,
                          bool need_sampler, void* workspace, size_t workspace_bytes,
                          std::vector<const MatParams*>& mps) {
  if (!mats || n_mats <= 0) return fail(NM_ERR_INVALID, "no materials");
  if (n_mats > 32) return fail(NM_ERR_UNSUPPORTED, "at most 32 materials per call");
  if (n >= (int64_t)1 << 31) return fail(NM_ERR_UNSUPPORTED, "batch too large for one call");
  if (!workspace || workspace_bytes < nm_multi_workspace_bytes(n, n_mats))
    return fail(NM_ERR_INVALID, "workspace too small (see nm_multi_workspace_bytes)");
  const int dev = mats[0]->device;
  mps.resize(n_mats);
  for (int k = 0; k < n_mats; ++k) {
    if (!mats[k]) return fail(NM_ERR_INVALID, "null material");
    if (mats[k]->device != dev) return fail(NM_ERR_INVALID, "materials on different devices");
    if (need_brdf && !mats[k]->mp.has_brdf) return fail(NM_ERR_INVALID, "material has no BRDF decoder");
    if (need_sampler && !mats[k]->mp.has_sampler) return fail(NM_ERR_INVALID, "material has no sampler decoder");
    mps[k] = &mats[k]->mp;
  }
  return NM_OK;
}

static int multi_binned_call(const std::vector<const MatParams*>& mps, int mode, const QueryArgs& a,
                             const int32_t* mat_id, int32_t multi_mode, void* workspace, void* stream,
                             int dev, const char* what) {
  DeviceGuard guard(dev);
  std::vector<int32_t> counts(mps.size());
  int32_t bad = 0;
  const cudaError_t e = multi_binned(mps.data(), (int32_t)mps.size(), mode, a, mat_id, workspace, counts.data(),
                                     &bad, multi_mode == NM_MULTI_BINNED, (cudaStream_t)stream);
  if (e == cudaErrorInvalidValue && bad) return fail(NM_ERR_INVALID, "mat_id out of range");
  return finish(nullptr, e, what);
}

int nm_eval_multi(const nm_material* const* mats, int32_t n_mats, int64_t n,
                  const int32_t* mat_id, const float* uv, const float* lod, int32_t lod_stride,
                  const float* u_rr, const float* wi, const float* wo, float* rgb_out,
                  int32_t mode, void* workspace, size_t workspace_bytes, void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!mat_id || !uv || !lod || !u_rr || !wi || !wo || !rgb_out)
    return fail(NM_ERR_INVALID, "null input");
  std::vector<const MatParams*> mps;
  int rc = multi_prologue(mats, n_mats, n, true, false, workspace, workspace_bytes, mps);
  if (rc != NM_OK) return rc;
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.wo = wo; a.rgb = rgb_out;
  const int dev = mats[0]->device;
  if (mode == NM_MULTI_BINNED || mode == NM_MULTI_BINNED_ASYNC)
    return multi_binned_call(mps, kModeEval, a, mat_id, mode, workspace, stream, dev, "nm_eval_multi(binned)");
  if (mode != NM_MULTI_DIVERGENT) return fail(NM_ERR_INVALID, "unknown multi-material mode");
  for (auto* m : mps)
    if (m->precise) return fail(NM_ERR_UNSUPPORTED, "divergent multi-material eval is fp16-path only");
  DeviceGuard guard(dev);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  MatParams* dev_mps = nullptr;
  if ((e = div_table(mps, mats, n_mats, dev, &dev_mps)) != cudaSuccess) return cuda_fail(e, "material table");
  return finish(nullptr, launch_eval_divergent(mps.data(), dev_mps, n_mats, mat_id, a, s),
                "nm_eval_multi(divergent)");
}

int nm_sample_pdf_multi(const nm_material* const* mats, int32_t n_mats, int64_t n, const int32_t* mat_id,
                        const float* uv, const float* lod, int32_t lod_stride, const float* u_rr,
                        const float* wi, const float* u3, float* wo_out, float* pdf_out, float* params9_out,
                        int32_t mode, void* workspace, size_t workspace_bytes, void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!mat_id || !uv || !lod || !u_rr || !wi || !u3 || !wo_out || !pdf_out)
    return fail(NM_ERR_INVALID, "null input");
  if (mode != NM_MULTI_BINNED && mode != NM_MULTI_BINNED_ASYNC)
    return fail(NM_ERR_UNSUPPORTED, "sample+pdf over several materials runs binned");
  std::vector<const MatParams*> mps;
  int rc = multi_prologue(mats, n_mats, n, false, true, workspace, workspace_bytes, mps);
  if (rc != NM_OK) return rc;
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.u3 = u3; a.ws = wo_out; a.pdf = pdf_out; a.params9 = params9_out;
  return multi_binned_call(mps, kModeSamplePdf, a, mat_id, mode, workspace, stream, mats[0]->device,
                           "nm_sample_pdf_multi");
}

int nm_query_multi(const nm_material* const* mats, int32_t n_mats, int64_t n, const int32_t* mat_id,
                   const float* uv, const float* lod, int32_t lod_stride, const float* u_rr, const float* wi,
                   const float* wo, const float* u3, float* rgb_out, float* ws_out, float* pdf_out,
                   int32_t mode, void* workspace, size_t workspace_bytes, void* stream) {
  NM_CHECK_N(n);
  if (n == 0) return NM_OK;
  if (!mat_id || !uv || !lod || !u_rr || !wi || !wo || !u3 || !rgb_out || !ws_out || !pdf_out)
    return fail(NM_ERR_INVALID, "null input");
  if (mode != NM_MULTI_BINNED && mode != NM_MULTI_BINNED_ASYNC)
    return fail(NM_ERR_UNSUPPORTED, "full queries over several materials run binned");
  std::vector<const MatParams*> mps;
  int rc = multi_prologue(mats, n_mats, n, true, true, workspace, workspace_bytes, mps);
  if (rc != NM_OK) return rc;
  QueryArgs a{};
  a.n = n; a.uv = uv; a.lod = lod; a.lod_stride = lod_stride ? 1 : 0; a.u_rr = u_rr;
  a.wi = wi; a.wo = wo; a.u3 = u3; a.rgb = rgb_out; a.ws = ws_out; a.pdf = pdf_out;
  return multi_binned_call(mps, kModeQuery, a, mat_id, mode, workspace, stream, mats[0]->device,
                           "nm_query_multi");
}

}  // extern "C"
