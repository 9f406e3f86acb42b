// nmq_internal.h — material layout shared by the host (nmq_abi.cu) and the
// kernels (nmq_kernels.cu).  Not part of the public ABI.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace nmq {

constexpr int kMaxLevels = 24;
constexpr int kMaxLayers = 16;
constexpr int kTile = 128;        // queries per MMA tile (M = 128, one per thread)
constexpr int kMaxWidth = 64;     // max padded layer width handled by the kernels
constexpr int kBiasCol = 504;     // TMEM column holding the shared [1,0..] bias chunk
constexpr int kTmemCols = 512;

struct LevelDesc {
  int32_t w, h;
  int64_t off;  // texel offset of the level in the latent buffer
};

// One MMA layer.  B operand (weights) lives in SMEM at `b_off` in the
// chunk-major K-major layout described in tc.cuh, N padded to n_pad rows.
//   first == 1: the input vector x (fan_in values + a 1.0 bias slot at
//               index fan_in) is written to TMEM as K = ksteps*16 fp16.
//   first == 0: input = previous layer's activation split hi/lo
//               (K = 2*in_pad) followed by the shared bias chunk (K = 16).
struct LayerDesc {
  uint32_t b_off;
  uint16_t n_pad;
  uint16_t in_pad;
  uint8_t ksteps;
  uint8_t first;
  uint8_t act;      // 0 linear, 1 leaky
  uint8_t out;      // true (unpadded) output width
  uint8_t precise;  // fp32 path: B = [W_hi | W_hi | W_lo] against A = [x_hi | x_lo | x_hi]
  uint16_t fan_in;  // true fan-in
  uint32_t w32_off; // float offset of the layer in MatParams::w32
};

struct MatParams {
  const uint4* latent;  // 16 B per texel (8 x fp16), or 32 B (8 x fp32) if texel_fp32
  int32_t n_levels;
  int32_t pow2;         // every level is a power of two in both dims
  int32_t texel_fp32;
  int32_t has_brdf, has_sampler;
  LevelDesc lv[kMaxLevels];
  const uint4* wblob;   // packed weights (global), copied to SMEM per CTA
  uint32_t wblob_bytes;
  int32_t use_frames, n_frames, albedo, isotropic;
  int32_t frame_layer;            // layer index or -1
  int32_t brdf_first, brdf_count; // layer range
  int32_t samp_first, samp_count;
  int32_t brdf_in;                // fan_in of the first BRDF layer (8 + 6*n_frames or 14)
  int32_t dmax;                   // max n_pad / in_pad over all layers (16/32/48/64)
  int32_t fast_arch;              // specialized pipelined kernel id (nmq_fast.cu), -1 = generic
  int32_t precise;                // fp32 path (generic kernel only)
  LayerDesc layers[kMaxLayers];
  // Specialized kernels (nmq_fast.cu) share one K=16 input chunk between the
  // frame layer, the sampler's first layer and the BRDF decoder's first
  // layer: chunk 0 = [z(8), wi(3), 1, 0 x 4], chunk 1 = [T.wi(6), T.wo(6), 0 x 4].
  // B operands re-packed for that K order (zero weights against wi where
  // the layer does not read it; bias against the 1 at K = 11):
  uint32_t fast_frame_off;  // frame layer, N = 16 (12 used), K = 16
  uint32_t fast_l1_off;     // BRDF first layer, N = hidden width, K = 32
  // fp32 copy (exact) of the BRDF output layer W -> 3|6, evaluated with packed
  // FFMA2 on the CUDA cores: ow[j][q] = (W[j][2q], W[j][2q+1]), ob[j]
  float2 ow[6][32];
  float ob[6];
  // fp32 copies (exact widenings of the fp16 weights) for the SIMT parts of
  // the exact-rounding path: the frame layer [W(8) | b] per
  // raw output (evaluated with the reference's sequential FMA order), and
  // every network in the reference's packed access order [w_row, bias] per
  // neuron (`w32` + LayerDesc::w32_off), read by the warp-cooperative
  // re-evaluation of queries whose decoder inputs round differently.
  float2 fw2[6][9];  // frame layer, both frames paired: (W[j][k], W[j + 6][k]), k = 8: bias
  const float* w32;
};

enum Mode : int {
  kModeFetch = 0,
  kModeEval = 1,       // fetch + eval
  kModeEvalZ = 2,      // eval from z
  kModeProxyZ = 3,     // infer_proxy from z
  kModeSamplePdf = 4,  // fetch + sampler + sample + pdf
  kModeQuery = 5,      // fetch + eval + sampler + sample + pdf
};

struct QueryArgs {
  int64_t n;
  const float* uv;
  const float* lod;
  int32_t lod_stride;
  const float* u_rr;
  const double* uv64;   // optional float64 coordinates (generic kernels): uv, lod, u_rr
  const double* lod64;
  const double* urr64;
  const float* z;
  const float* wi;
  const float* wo;
  const double* wi64;   // optional float64 directions (generic kernels; wi / wo then unused)
  const double* wo64;
  const float* u3;
  const int32_t* idx;   // optional input-row gather: row i of the launch reads query idx[i]
                        // (i counted from the segment base, like out_idx)
  const int32_t* out_idx;  // optional output rows: results of row i go to row out_idx[i]
                           // (binned multi-material writes straight to query order)
  const int32_t* seg;      // optional device {base, count}: the launch covers input rows
                           // [base, base + count) (n is then only a capacity bound);
                           // lets binned segments launch without a host round trip
  int32_t max_ctas;        // optional cap on the persistent grid (0 = one CTA per SM):
                           // concurrent segment launches on disjoint SM subsets
  float* rgb;
  float* albedo;
  float* ws;
  float* pdf;
  float* params9;
  float* z_out;
  int32_t* level;
  int32_t* taps;
  float* wts;
  int32_t spp_log2;   // eval with img: per-pixel mean over 2^spp_log2 consecutive rows (in-kernel)
  float* img;          // (n >> spp_log2, 3), accumulated (zeroed by the caller)
  int32_t trilinear;  // fetch: deterministic trilinear filtering instead of the roulette pick
  float* dbg;  // fast kernel calibration dump: fp32 T.wi, T.wo and frame conditioning (14 floats/row)
};

// pipelined tcgen05 kernels (nmq_fast.cu); cudaErrorNotSupported = not
// applicable, use the generic kernel
cudaError_t launch_fast(const MatParams& mp, int mode, const QueryArgs& a, cudaStream_t s);
// scale of the leaky-ReLU trick shared by the specialized kernels: c = 1 + k
constexpr double kLeakyScale = 1.0 + 0.98019802570343017578;
// launchers (nmq_kernels.cu); return cudaError_t of the launch
cudaError_t launch_fused(const MatParams& mp, int mode, const QueryArgs& a, cudaStream_t s,
                         int groups_override = 0);
// the decoder's fp16 direction inputs in the reference's arithmetic (tw_exact), one row per thread
cudaError_t launch_decoder_inputs(const MatParams& mp, int64_t n, const float* z, const float* wi,
                                  const float* wo, const double* wi64, const double* wo64, uint32_t* x16,
                                  cudaStream_t s);
cudaError_t launch_fetch(const MatParams& mp, const QueryArgs& a, cudaStream_t s);
cudaError_t launch_sample(int64_t n, const float* p9, const float* wi, const float* u3,
                          float* wo, cudaStream_t s);
cudaError_t launch_pdf(int64_t n, const float* p9, const float* wi, const float* wo, float* pdf,
                       cudaStream_t s);
// multi-material (nmq_multi.cu / nmq_kernels.cu)
size_t multi_workspace_bytes(int64_t n, int32_t n_mats);
cudaError_t multi_binned(const MatParams* const* mps, int32_t n_mats, int mode, const QueryArgs& a,
                         const int32_t* mat_id, void* ws, int32_t* host_counts, int32_t* bad,
                         bool checked, cudaStream_t s);
cudaError_t launch_eval_divergent(const MatParams* const* mps_host, const MatParams* mps_dev,
                                  int32_t n_mats, const int32_t* mat_id, const QueryArgs& a,
                                  cudaStream_t s);
int smem_bytes_for(const MatParams& mp);
// training-side kernels (nmq_train.cu)
cudaError_t launch_texel_grads(const MatParams& mp, int64_t n, const float* uv, const int32_t* level,
                               const float* z_grad, float* grad, cudaStream_t s);
cudaError_t launch_mlp_forward(const int32_t* fi, const int32_t* fo, const int32_t* act, int n_layers,
                               const float* wts, int32_t w_floats, int64_t B, const float* x,
                               float* x_cache, float* pre_cache, float* out, cudaStream_t s);
cudaError_t launch_mlp_backward(const int32_t* fi, const int32_t* fo, const int32_t* act, int n_layers,
                                const float* wts, int32_t w_floats, int64_t B, const float* x_cache,
                                const float* pre_cache, const float* out_grad, double* g_cache,
                                double* dparams, double* dx, cudaStream_t s);
// KL sampler-loss heads (nmq_kl.cu)
cudaError_t launch_kl_sample(int64_t b, int frames, int nf, int iso, const float* raw_s,
                             const float* raw_f, const float* z, const double* wi, const double* u_d,
                             const double* u_s, float* x2, double* scr, cudaStream_t st);
cudaError_t launch_kl_target(int64_t b, int out_w, const float* y, const double* scr, double* tgt,
                             double* lum, float* og, cudaStream_t st);
cudaError_t launch_kl_target_dir(int64_t b, int frames, int nf, const float* raw_f, const double* dx,
                                 const double* scr, const double* lum, double* dtgt, cudaStream_t st);
cudaError_t launch_kl_grad(int64_t b, int iso, const float* raw_s, const double* wi, const double* scr,
                           const double* tgt, const double* dtgt, float* draw, double* loss_rows,
                           cudaStream_t st);
// level of detail from ray cones (nmq_lod.cu)
cudaError_t launch_footprint_level(int64_t n, const double* area, int32_t n_levels, double* out,
                                   cudaStream_t s);
cudaError_t launch_cone_level(int64_t n, const float* cone_w, const float* cone_s, const float* t,
                              const float* cos_hit, const float* density, int32_t density_stride,
                              int32_t n_levels, float* lod, cudaStream_t s);
// Raise a kernel's dynamic shared memory limit to the device maximum, once
// per kernel (thread-safe; a per-launch set-then-launch pair would race with
// another host thread lowering the limit in between).  Returns the limit
// (bytes of dynamic SMEM available to the kernel) or -1 on failure.
int max_dynamic_smem(const void* kernel);
extern std::atomic<int64_t> g_launches;  // host threads may launch concurrently
// kernel path: 0 = auto (tcgen05 pipelined, then generic), 1 = generic only,
// 2 = tcgen05 pipelined (falls back to generic)
extern int g_kernel_path;
extern float g_tw_margin;  // nm_set_tw_margin (<= 0: built-in bound)
extern std::atomic<int> g_last_path;  // family of the last launch_fused (1/2 as above)

}  // namespace nmq
