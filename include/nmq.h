/*
 * nmq.h — C ABI of the B200 (sm_100a) neural-material query library
 * (libnmq.so).  This is the drop-in boundary for the query hot path of the
 * reference `neuralmat` package (arXiv 2305.02678 "Real-Time Neural
 * Appearance Models").  Every entry point below replaces one reference
 * function; the reference file:line is cited on each (paths relative to
 * /root/reference/pkg/src/neuralmat).
 *
 * Conventions
 *  - All array arguments of the query entry points are DEVICE pointers on the
 *    material's device, fp32 (or int32), C-contiguous, batch-first:
 *    uv (n,2), lod (n,) or scalar, u_rr (n,), wi/wo (n,3), u3 (n,3),
 *    z (n,8), params9 (n,9), rgb/albedo/ws (n,3), pdf (n,), level (n,).
 *  - `stream` is a cudaStream_t passed as void*.  Launches are asynchronous;
 *    many streams may launch on one material at once.  Allocation: the
 *    device-pointer entry points allocate nothing per call, except one
 *    grow-only scratch buffer per (device, stream) — the fp16 fast path's
 *    exact-rounding queue (stream-ordered cudaMallocAsync, reused by every
 *    later call on that stream).  nm_eval_host keeps one grow-only device
 *    staging buffer per device (cudaMalloc when a call needs more; calls on
 *    one device serialize on it).
 *    Nothing is freed before nm_destroy / process exit.
 *  - Optional outputs may be NULL.  `lod_stride` is 1 for a per-query array
 *    and 0 to broadcast lod[0] (the reference's scalar level, latent.py:91).
 *  - Return value: 0 = ok, < 0 = error; nm_last_error() returns a
 *    thread-local message for the last failing call on this thread.
 *  - The material handle is immutable after creation.
 *
 * Parameter block `params9` (the renderer's per-vertex cache,
 * render.py:370-372): wd, ws, mu_d.x, mu_d.y, alpha.x, alpha.y, rho,
 * mu_s.x, mu_s.y with the alpha floor and rho clamp already applied
 * (proxy.py:42-50).
 */
#ifndef NMQ_H
#define NMQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NMQ_VERSION 1

enum nm_status {
  NM_OK = 0,
  NM_ERR_INVALID = -1,  /* bad argument / shape (reference raises ValueError) */
  NM_ERR_CUDA = -2,     /* CUDA runtime failure */
  NM_ERR_UNSUPPORTED = -3 /* architecture outside what the kernels implement */
};

enum nm_act { NM_ACT_LINEAR = 0, NM_ACT_LEAKY = 1 }; /* mlp.py:22 _ACT_CODES */

/* DIVERGENT: mixed tiles decoded directly; BINNED: sort into per-material
 * segments, coherent kernel per segment, ids validated (one host round trip);
 * BINNED_ASYNC: the same without the host round trip (segment sizes stay on
 * the device; rows with out-of-range ids are left untouched). */
/* nm_query_f64 modes */
enum nm_query_mode { NM_QUERY_EVAL = 0, NM_QUERY_SAMPLE_PDF = 1, NM_QUERY_FULL = 2 };

enum nm_multi_mode { NM_MULTI_DIVERGENT = 0, NM_MULTI_BINNED = 1, NM_MULTI_BINNED_ASYNC = 2 };

/* One quantized network exactly as the reference holds it
 * (QuantizedMlp, mlp.py:165-233): per layer, per output neuron,
 * [w_row(fan_in) ..., bias] as IEEE fp16 bits, layers back to back. */
typedef struct nm_net_desc {
  int32_t n_layers;
  const int32_t* fan_in;  /* [n_layers] */
  const int32_t* fan_out; /* [n_layers] */
  const int32_t* act;     /* [n_layers] nm_act */
  const uint16_t* packed; /* fp16 bits, host memory */
  /* fp32 master weights in the same access order (Mlp.layers, mlp.py:50-69);
   * required when the material is created with precise = 1 */
  const float* weights;
} nm_net_desc;

/* Everything NeuralMaterial.half() produces (neural.py:147-161). */
typedef struct nm_material_desc {
  int32_t channels;          /* latent channels; must be 8 (latent.py:17) */
  int32_t use_frames;        /* NeuralMaterialConfig.use_frames */
  int32_t n_frames;          /* learned shading frames (neural.py:30) */
  int32_t albedo_head;       /* BRDF decoder emits 6 outputs */
  int32_t sampler_isotropic; /* sampler emits 2 outputs (neural.py:319) */
  /* A network with n_layers == 0 is absent; a material with no BRDF and no
   * sampler network is latent-only (nm_fetch works, the decoders fail). */
  nm_net_desc frame;         /* ignored when use_frames == 0 */
  nm_net_desc brdf;
  nm_net_desc sampler;
  int32_t width, height;     /* level-0 latent resolution */
  int32_t n_levels;          /* must equal the max(1, w//2) chain length */
  const void* latent;        /* levels back to back, (H,W,C) each: fp16 bits,
                                or fp32 when latent_fp32 = 1 */
  int32_t latent_fp32;       /* texels are 8 x fp32 (32 B) instead of 8 x fp16 */
  int32_t latent_on_device;  /* 1: `latent` is a device pointer on `device` */
  /* 1: the reference's fp32 path (fp16=False: Mlp.forward on fp32 master
   * weights, neural.py:288-293, 357-360): inputs, hidden activations and
   * weights each carried as an fp16 (hi, lo) pair on the tensor cores
   * (W_hi x_hi + W_hi x_lo + W_lo x_hi), fp32 accumulation; pair with the
   * fp32 master pyramid (latent_fp32 = 1).  0: the fp16 inference path. */
  int32_t precise;
} nm_material_desc;

typedef struct nm_material nm_material;

typedef struct nm_material_info {
  int32_t device;
  int32_t n_levels;
  int64_t latent_texels;     /* texels over all levels */
  int64_t latent_bytes;
  int32_t weight_bytes;      /* packed MMA-layout weights staged per CTA */
  int32_t brdf_width;        /* padded max hidden width of the BRDF decoder */
  int32_t sampler_width;
} nm_material_info;

/* --- material lifetime (replaces NeuralMaterial.half() caching,
 *     neural.py:147-161, and load-time upload) --------------------------- */
int nm_material_create(const nm_material_desc* desc, int device, nm_material** out);
int nm_material_destroy(nm_material* mat);
int nm_material_info_get(const nm_material* mat, nm_material_info* info);
/* level table: w, h per level and texel offset of each level (n_levels each) */
int nm_material_levels(const nm_material* mat, int32_t* w, int32_t* h, int64_t* offset);
/* device pointer to the fp16 texels (read-only; for tests / LoD tooling) */
const void* nm_material_latent_ptr(const nm_material* mat);

/* --- latent fetch: LatentPyramid.fetch (latent.py:84-98) with
 *     choose_level (:76-82) and _taps (:56-74).  taps_out (n,4,2) int32
 *     (x,y) and wts_out (n,4) are debug outputs mirroring _taps. --------- */
int nm_fetch(const nm_material* mat, int64_t n, const float* uv, const float* lod,
             int32_t lod_stride, const float* u_rr, float* z_out, int32_t* level_out,
             int32_t* taps_out, float* wts_out, void* stream);

/* --- eval_material (neural.py:303-309): fetch + frames + BRDF decoder +
 *     brdf_output + horizon mask, fused (the coherent eval kernel). ------- */
/* float64 coordinates (uv (n,2), lod, u_rr), the reference's own dtype
 * (latent.py:59-82 computes in float64; render.py:369 passes float64): level
 * pick, taps and weights exactly as numpy does them, so levels / taps / z stay
 * bit-exact for any float64 input (the fp32 entry points are exact for
 * fp32-representable inputs).  nm_query_f64 also takes the directions in
 * float64 (wi, wo (n,3); wo unused by NM_QUERY_SAMPLE_PDF): the decoder's
 * T.wi / T.wo are formed from them in float64 as the reference does
 * (neural.py:280-287); the sampler input and the proxy use them narrowed to
 * fp32 (neural.py:358 `astype(np.float32)`).  Runs on the generic kernels. */
int nm_fetch_f64(const nm_material* m, int64_t n, const double* uv, const double* lod, int32_t lod_stride,
                 const double* u_rr, float* z_out, int32_t* level_out, int32_t* taps_out, float* wts_out,
                 void* stream);
int nm_query_f64(const nm_material* m, int32_t mode, int64_t n, const double* uv, const double* lod,
                 int32_t lod_stride, const double* u_rr, const double* wi, const double* wo, const float* u3,
                 float* rgb_out, float* albedo_out, float* ws_out, float* pdf_out, float* params9_out,
                 int32_t* level_out, void* stream);
/* Eval reduced to the per-pixel sample mean in the kernel epilogue (the
 * renderer's spp accumulation, render.py:565): rows are pixel * spp + s,
 * spp a power of two, n a multiple of spp; img_out (n / spp, 3) fp32 is
 * overwritten.  Per-sample rgb never reaches memory. */
int nm_eval_spp(const nm_material* m, int64_t n, const float* uv, const float* lod, int32_t lod_stride,
                const float* u_rr, const float* wi, const float* wo, int32_t spp, float* img_out, void* stream);
/* Deterministic trilinear fetch (optional filtering mode; the reference only
 * states it as the roulette fetch's expectation, latent.py:84-92, checked in
 * tests/test_acceptance.py:242-255): z = (1 - f) bilinear(floor l) +
 * f bilinear(ceil l), l clipped to [0, L-1], in float64 from the two float32
 * bilinear fetches (latent.py:100-107), narrowed to fp32.  level_out
 * (nullable) receives floor(l). */
int nm_fetch_trilinear(const nm_material* m, int64_t n, const float* uv, const float* lod,
                       int32_t lod_stride, float* z_out, int32_t* level_out, void* stream);
int nm_eval(const nm_material* mat, int64_t n, const float* uv, const float* lod,
            int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
            float* rgb_out, float* albedo_out, int32_t* level_out, void* stream);

/* --- eval_brdf (neural.py:273-300), fp16 path, from given latent codes -- */
int nm_eval_z(const nm_material* mat, int64_t n, const float* z, const float* wi,
              const float* wo, float* rgb_out, float* albedo_out, void* stream);
/* eval_brdf on the reference's float64 directions (render.py passes float64;
 * T.wi / T.wo formed from them in float64, neural.py:280-287). */
int nm_eval_z_f64(const nm_material* m, int64_t n, const float* z, const double* wi, const double* wo,
                  float* rgb_out, float* albedo_out, void* stream);
/* Check hook for the exact-rounding contract: the BRDF decoder's direction
 * inputs exactly as the reference rounds them (neural.py:282-287: frames
 * from the frame layer's fp32 outputs, T.wi / T.wo in float64 with numpy's
 * operation order, then fp32, then fp16).  x16_out (n, 12) fp16 bit patterns
 * [T.wi (3 per frame), T.wo (3 per frame)] (one frame: 6 values, then 0).
 * z (n, 8) fp32 holding fp16 values; directions fp32 (wi, wo) or float64
 * (wi64, wo64; then wi / wo may be NULL).  fp16 materials with frames. */
int nm_decoder_inputs(const nm_material* m, int64_t n, const float* z, const float* wi, const float* wo,
                      const double* wi64, const double* wo64, uint16_t* x16_out, void* stream);

/* --- infer_proxy (neural.py:353-362) + proxy_from_raw (:317-331) -------- */
int nm_infer_proxy(const nm_material* mat, int64_t n, const float* z, const float* wi,
                   float* params9_out, void* stream);

/* --- proxy.sample (proxy.py:168-180) and proxy.pdf (proxy.py:129-135) on
 *     a params9 block (no material needed). ------------------------------ */
int nm_sample(int64_t n, const float* params9, const float* wi, const float* u3,
              float* wo_out, void* stream);
int nm_pdf(int64_t n, const float* params9, const float* wi, const float* wo, float* pdf_out,
           void* stream);

/* --- fused sampling path: fetch + sampler decoder + proxy + sample + pdf of
 *     the sampled direction (render.py:368-372 + 401-402). --------------- */
int nm_sample_pdf(const nm_material* mat, int64_t n, const float* uv, const float* lod,
                  int32_t lod_stride, const float* u_rr, const float* wi, const float* u3,
                  float* ws_out, float* pdf_out, float* params9_out, int32_t* level_out,
                  void* stream);

/* --- one full query: one fetch feeding eval(wi, wo) and the sampler;
 *     ws = sample(u3), pdf(ws). ------------------------------------------ */
int nm_query(const nm_material* mat, int64_t n, const float* uv, const float* lod,
             int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
             const float* u3, float* rgb_out, float* ws_out, float* pdf_out,
             int32_t* level_out, void* stream);

/* --- multi-material eval (render.py:352-356 groups by material):
 *     mat_id (n,) int32 in [0, n_mats).  DIVERGENT decodes mixed tiles
 *     directly; BINNED first bins queries by material with warp-aggregated
 *     counting, then runs the coherent kernel per bin.  workspace must hold
 *     nm_multi_workspace_bytes(n, n_mats) bytes of device memory.  Host
 *     blocking: BINNED waits for the bin counts (one D2H, to validate ids
 *     and size the per-bin launches); BINNED_ASYNC never waits; DIVERGENT
 *     waits only on the first call with a given material list (its device
 *     table of parameter blocks is uploaded once and cached until one of
 *     the materials is destroyed). --------------------------------------- */
size_t nm_multi_workspace_bytes(int64_t n, int32_t n_mats);
int nm_eval_multi(const nm_material* const* mats, int32_t n_mats, int64_t n,
                  const int32_t* mat_id, const float* uv, const float* lod,
                  int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
                  float* rgb_out, int32_t mode, void* workspace, size_t workspace_bytes,
                  void* stream);
/* The renderer's per-vertex material groups for the sampler side
 * (render.py:361-372, 391-409): sample + pdf, and the full query (eval +
 * sample + pdf), each row with its own material mats[mat_id[i]].  Binned
 * modes only (NM_MULTI_BINNED / NM_MULTI_BINNED_ASYNC; DIVERGENT returns
 * NM_ERR_UNSUPPORTED).  Same workspace as nm_eval_multi. */
int nm_sample_pdf_multi(const nm_material* const* mats, int32_t n_mats, int64_t n, const int32_t* mat_id,
                        const float* uv, const float* lod, int32_t lod_stride, const float* u_rr,
                        const float* wi, const float* u3, float* wo_out, float* pdf_out, float* params9_out,
                        int32_t mode, void* workspace, size_t workspace_bytes, void* stream);
int nm_query_multi(const nm_material* const* mats, int32_t n_mats, int64_t n, const int32_t* mat_id,
                   const float* uv, const float* lod, int32_t lod_stride, const float* u_rr, const float* wi,
                   const float* wo, const float* u3, float* rgb_out, float* ws_out, float* pdf_out,
                   int32_t mode, void* workspace, size_t workspace_bytes, void* stream);

/* --- misc -------------------------------------------------------------- */
/* nm_eval with HOST buffers; blocking (the outputs are complete on return),
 * ordered after prior work on `stream`.  albedo_out (n,3) and level_out (n,)
 * are optional.  All buffers pinned (page-locked): zero-copy, one fused
 * launch reading the inputs and writing the outputs over PCIe (`chunk`
 * unused; env NMQ_HOST_ZEROCOPY=0 disables).  Otherwise the batch
 * streams through device staging in `chunk`-query pieces (0 = 512k): one
 * stream for the H2D copies, one for the kernels, one for the D2H copies.
 * The reference call it replaces is eval_material on numpy arrays
 * (neural.py:303). */
int nm_eval_host(const nm_material* mat, int64_t n, const float* uv, const float* lod,
                 int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
                 float* rgb_out, float* albedo_out, int32_t* level_out, int64_t chunk, void* stream);

/* eval_material's own call shape on host buffers (neural.py:303-309): the
 * reference's output dtypes — colours (n,3) and albedo float64, levels
 * int64 — widened on the device, so the host never converts.  Pageable
 * buffers stream through a pinned bounce pipeline: a pool of host threads
 * (NMQ_HOST_THREADS, default min(8, hardware threads)) copies each chunk of
 * inputs into a pinned slot and each chunk of results out of one, the copy
 * engines move the pinned slots, chunks of `chunk` queries (0 = 256k)
 * overlap over 4 slots; page-locked result buffers receive the DMA
 * directly.  Blocking.  nm_eval_host's pageable path uses the
 * same pipeline (NMQ_HOST_BOUNCE=0: the driver's own staging). */
int nm_eval_host_ref(const nm_material* m, int64_t n, const float* uv, const float* lod, int32_t lod_stride,
                     const float* u_rr, const float* wi, const float* wo, double* rgb_out, double* albedo_out,
                     int64_t* level_out, int64_t chunk, void* stream);

/* Training-side kernels (device pointers, async on `stream`).
 *  nm_texel_grads: exact adjoint of the fetch (latent.py:109-119
 *    accumulate_texel_grads): z_grad (n, 8) scattered onto the four bilinear
 *    taps of each query at its level (int32) and ADDED into grad_texels
 *    (texels, 8) fp32, laid out like the material's latent (levels back to back).
 *  nm_mlp_*: the fp32 network engine (mlp.py:90-116).  forward_cached runs
 *    the batch (x (B, in) -> out (B, out)) keeping what backward needs in
 *    `cache` (nm_mlp_cache_bytes); backward writes d(sum(out * out_grad)) /
 *    d(params) into dparams (float64, the weights' access order [dW_row, db]
 *    per neuron per layer, overwritten) and dx (B, in) float64. */
typedef struct nm_mlp nm_mlp;
int nm_texel_grads(const nm_material* mat, int64_t n, const float* uv, const int32_t* level,
                   const float* z_grad, float* grad_texels, void* stream);
int nm_mlp_create(const nm_net_desc* net, int device, nm_mlp** out);
int nm_mlp_set_weights(nm_mlp* mlp, const float* weights);
int nm_mlp_destroy(nm_mlp* mlp);
int32_t nm_mlp_params(const nm_mlp* mlp);
size_t nm_mlp_cache_bytes(const nm_mlp* mlp, int64_t batch);
int nm_mlp_forward_cached(const nm_mlp* mlp, int64_t batch, const float* x, float* out, void* cache,
                          void* stream);
int nm_mlp_backward(const nm_mlp* mlp, int64_t batch, void* cache, const float* out_grad,
                    double* dparams, double* dx, void* stream);

/* KL sampler loss (replaces the heads of training.sampler_loss_and_grads,
 * training.py:219-273, and its default target _brdf_target_and_grad,
 * training.py:187-216; the three network passes run on nm_mlp_*).  Row
 * layouts, all device pointers, b = batch:
 *   nm_kl_sample: raw_s (b, 9 | 2 isotropic) sampler outputs, raw_f (b, 6 nf)
 *     frame-layer outputs (ignored without frames), z (b, 8), wi (b, 3) f64,
 *     u_d / u_s (b, 2) f64 -> x2 (2b, in) fp32 BRDF decoder inputs at the
 *     diffuse (rows [0, b)) and specular (rows [b, 2b)) samples, in = 8 + 6 nf
 *     (14 without frames); scratch (b, NM_KL_SCRATCH) f64 (samples + aux).
 *   nm_kl_target: y (2b, out_w) decoder outputs -> target (2b) = lum(f) cos + 1e-4,
 *     lum (2b), out_grad (2b, out_w) fp32 = d target / d y (columns >= 3 zero).
 *   nm_kl_target_dir: dx (2b, in) f64 decoder-input gradients -> dtarget (2b, 3).
 *   nm_kl_grad: target / dtarget (2b ...) -> draw (b, 9 | 2) fp32 = d loss / d raw
 *     (the batch mean's 1/b included), loss_rows (b) f64 (loss = their mean). */
#define NM_KL_SCRATCH 17
int nm_kl_sample(int64_t b, int32_t use_frames, int32_t n_frames, int32_t isotropic, const float* raw_s,
                 const float* raw_f, const float* z, const double* wi, const double* u_d,
                 const double* u_s, float* x2_out, double* scratch, void* stream);
int nm_kl_target(int64_t b, int32_t out_w, const float* y, const double* scratch, double* target_out,
                 double* lum_out, float* out_grad, void* stream);
int nm_kl_target_dir(int64_t b, int32_t use_frames, int32_t n_frames, const float* raw_f,
                     const double* dx, const double* scratch, const double* lum, double* dtarget_out,
                     void* stream);
int nm_kl_grad(int64_t b, int32_t isotropic, const float* raw_s, const double* wi,
               const double* scratch, const double* target, const double* dtarget, float* draw_out,
               double* loss_rows, void* stream);

/* Level of detail from ray cones (replaces render.footprint_to_level,
 * render.py:334-337, and the footprint in render._surface_frames_and_level,
 * render.py:436-443).  float64 like the reference.
 *   nm_footprint_level: level = clip(0.5 log2(max(area, 1)), 0, n_levels-1)
 *   nm_cone_level:      area = ((w + s t) / max(|cos_hit|, 0.05) * density)^2,
 *                       level as above, rounded to the fp32 lod the query
 *                       entry points take; density_stride 0 = one density. */
int nm_footprint_level(int64_t n, const double* area_texels, int32_t n_levels, double* level_out,
                       void* stream);
int nm_cone_level(int64_t n, const float* cone_w, const float* cone_s, const float* t,
                  const float* cos_hit, const float* density, int32_t density_stride,
                  int32_t n_levels, float* lod_out, void* stream);

const char* nm_last_error(void);
int nm_version(void);
/* number of fused-kernel launches issued by this process (for bench claims) */
int64_t nm_launch_count(void);
/* test hook: 0 = auto (default: the pipelined tcgen05 kernels for materials
 * matching a specialized architecture), 1 = always the runtime-generic
 * kernel, 2 = pipelined tcgen05 (falls back to the generic kernel when
 * inapplicable) */
int nm_set_kernel_path(int path);
/* which kernel family ran the last query launch of this process:
 * 1 = generic, 2 = pipelined tcgen05 */
int nm_last_kernel_path(void);
/* test hook of the exact-rounding path: error bound, per unit
 * frame conditioning, under which the pipelined kernels queue a row's fp16
 * direction inputs for exact resolution.  <= 0 restores the built-in bound;
 * a huge value queues every above-horizon row (exercises the resolve path). */
int nm_set_tw_margin(float delta);
/* calibration dump of the pipelined eval kernel: like nm_eval (fp16 path),
 * plus per row its fp32 fast-path [T.wi(6), T.wo(6)] and the two frames'
 * conditioning factors (14 floats per row) */
int nm_eval_debug_tw(const nm_material* m, int64_t n, const float* uv, const float* lod,
                     int32_t lod_stride, const float* u_rr, const float* wi, const float* wo,
                     float* rgb_out, float* dbg_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NMQ_H */
