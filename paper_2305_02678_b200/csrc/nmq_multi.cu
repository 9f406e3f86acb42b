// nmq_multi.cu — multi-material queries (reference: render.py:352-356 groups
// the hits of one path vertex by material and runs each group through its
// own network).  Two execution modes, as in the paper:
//
//  * BINNED: queries are binned by material id with warp-aggregated
//    counting (__match_any_sync + __popc, one atomic per distinct id per
//    warp), an exclusive scan, and a warp-aggregated scatter that permutes
//    the inputs into contiguous per-material segments (16-byte aligned); the
//    coherent fused kernel then runs once per segment and writes each result
//    straight to its query's row (output-row indirection, no scatter-back
//    pass).
//  * DIVERGENT: no reordering; every 128-query tile loops over the
//    materials present in it and decodes the whole tile with each of them,
//    keeping each row's own material (nmq_kernels.cu, kModeEvalMulti).
#include <cstdint>
#include <mutex>
#include "nmq_internal.h"

namespace nmq {
namespace {

constexpr int kMaxMats = 64;

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per-material counts.  Up to 8 materials: per-thread register counters
// over a grid-stride loop, warp sums (__reduce_add_sync), one shared atomic
// per material per warp and one global atomic per material per CTA (few
// CTAs: global atomics on a handful of counters serialise at L2).  More
// materials: warp-aggregated shared atomics (__match_any_sync).
__global__ void __launch_bounds__(256) bin_count_kernel(int64_t n, int32_t n_mats,
                                                        const int32_t* __restrict__ mat_id,
                                                        int32_t* __restrict__ counts,
                                                        int32_t* __restrict__ bad) {
  __shared__ int32_t sc[kMaxMats];
  for (int i = threadIdx.x; i < n_mats; i += blockDim.x) sc[i] = 0;
  __syncthreads();
  if (n_mats <= 8) {
    int32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool b = false;
    auto add = [&](int m) {
      b |= m < 0 || m >= n_mats;
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] += m == k;
    };
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = ((uintptr_t)mat_id & 15u) == 0 ? n / 4 : 0;  // 16-byte loads
    for (int64_t j = gt; j < n4; j += gs) {
      const int4 v = __ldg(reinterpret_cast<const int4*>(mat_id) + j);
      add(v.x);
      add(v.y);
      add(v.z);
      add(v.w);
    }
    for (int64_t i = 4 * n4 + gt; i < n; i += gs) add(__ldg(mat_id + i));
    if (b) atomicExch(bad, 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int32_t w = __reduce_add_sync(0xffffffffu, c[k]);
      if ((threadIdx.x & 31) == 0 && k < n_mats && w) atomicAdd(&sc[k], w);
    }
  } else {
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = base + threadIdx.x;
      const bool in = i < n;
      int m = in ? __ldg(mat_id + i) : -1;
      if (in && (m < 0 || m >= n_mats)) {
        atomicExch(bad, 1);
        m = -1;
      }
      const uint32_t active = __ballot_sync(0xffffffffu, m >= 0);
      if (m >= 0) {
        const uint32_t peers = __match_any_sync(active, m);
        if ((peers & lanemask_lt()) == 0) atomicAdd(&sc[m], __popc(peers));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_mats; i += blockDim.x)
    if (sc[i]) atomicAdd(counts + i, sc[i]);
}

// Each CTA bins a chunk of kScatterRows queries: ranks within the chunk per
// material from warp-aggregated SHARED atomics, ONE global atomic per
// material per CTA reserves the chunk's contiguous range of each segment
// (one global atomic per distinct id per warp — 5 x 65k atomics on 5
// counters for C4 — serialised at L2: 115 us per 2.07M queries).  The
// chunk's inputs are staged into SMEM in input order with coalesced 16-byte
// loads (every array of a chunk is one contiguous range), and written out in
// segment order — position p of the chunk's sorted order reads its source
// row from SMEM — so every segment range is written with coalesced stores.
// Ids outside [0, n_mats) are skipped (bin_count_kernel flags them).
constexpr int kScatterItems = 2;  // 512 rows: 18..32 KB SMEM, full occupancy
constexpr int kScatterRows = 256 * kScatterItems;
// SMEM of one chunk: src[R] | uv[2R] urr[R] wi[3R] | lod[R] | wo[3R] | u3[3R]
// (the optional arrays only when present; gather mode: src only)
__host__ __device__ constexpr size_t scatter_smem_bytes(bool gather, bool lod_arr, bool has_wo, bool has_u3) {
  return gather ? (size_t)kScatterRows * 4
                : (size_t)kScatterRows * 4 * (7 + (lod_arr ? 1 : 0) + (has_wo ? 3 : 0) + (has_u3 ? 3 : 0));
}

// count floats from src into SMEM dst with 16-byte loads when both ends allow
__device__ __forceinline__ void stage_floats(float* dst, const float* __restrict__ src, int count) {
  if ((((uintptr_t)src) & 15u) == 0 && (count & 3) == 0) {
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll 4
    for (int i = threadIdx.x; i < count / 4; i += blockDim.x) d4[i] = __ldg(s4 + i);
  } else {
    for (int i = threadIdx.x; i < count; i += blockDim.x) dst[i] = __ldg(src + i);
  }
}

__global__ void __launch_bounds__(256) bin_scatter_kernel(
    int64_t n, int32_t n_mats, const int32_t* __restrict__ mat_id, const int32_t* __restrict__ counts,
    int32_t* __restrict__ seg, int32_t* __restrict__ cursor,
    int32_t* __restrict__ order, const float* __restrict__ uv, const float* __restrict__ lod,
    int32_t lod_stride, const float* __restrict__ urr, const float* __restrict__ wi,
    const float* __restrict__ wo, const float* __restrict__ u3, float* __restrict__ p_uv,
    float* __restrict__ p_lod, float* __restrict__ p_urr, float* __restrict__ p_wi, float* __restrict__ p_wo,
    float* __restrict__ p_u3) {
  extern __shared__ __align__(16) float sm_f[];
  struct {
    float *uv, *urr, *wi, *lod, *wo, *u3;
    int32_t* src;
  } S;
  {
    float* q = sm_f;
    S.src = reinterpret_cast<int32_t*>(q); q += kScatterRows;
    S.uv = q; q += 2 * kScatterRows;
    S.urr = q; q += kScatterRows;
    S.wi = q; q += 3 * kScatterRows;
    S.lod = q; if (lod_stride) q += kScatterRows;
    S.wo = q; if (wo) q += 3 * kScatterRows;
    S.u3 = q;
  }
  __shared__ int32_t cnt[kMaxMats], loc[kMaxMats + 1], base[kMaxMats], off[kMaxMats];
  for (int i = threadIdx.x; i < n_mats; i += blockDim.x) cnt[i] = 0;
  if (threadIdx.x == 0) {
    // segment bases: exclusive scan of the counts, padded to multiples of 4
    // rows so every segment's staged inputs are 16-byte aligned (TMA); CTA 0
    // publishes {base, count} per segment for the segment launches
    int32_t acc = 0;
    for (int m = 0; m < n_mats; ++m) {
      const int32_t c = counts[m];
      off[m] = acc;
      if (blockIdx.x == 0) {
        seg[2 * m] = acc;
        seg[2 * m + 1] = c;
      }
      acc += (c + 3) & ~3;
    }
  }
  const int64_t c0 = (int64_t)blockIdx.x * kScatterRows;
  const int rows = (int)(n - c0 < kScatterRows ? n - c0 : kScatterRows);
  int mi[kScatterItems];
#pragma unroll
  for (int k = 0; k < kScatterItems; ++k) {
    const int r = k * 256 + threadIdx.x;
    mi[k] = r < rows ? __ldg(mat_id + c0 + r) : -1;
  }
  const bool gather = p_uv == nullptr;  // only the row order (segments gather their inputs)
  if (!gather) {  // the chunk's inputs, input order (in flight together with the ids)
    stage_floats(S.uv, uv + 2 * c0, 2 * rows);
    if (lod_stride) stage_floats(S.lod, lod + c0, rows);
    stage_floats(S.urr, urr + c0, rows);
    stage_floats(S.wi, wi + 3 * c0, 3 * rows);
    if (wo) stage_floats(S.wo, wo + 3 * c0, 3 * rows);
    if (u3) stage_floats(S.u3, u3 + 3 * c0, 3 * rows);
  }
  __syncthreads();
  int32_t rk[kScatterItems];
#pragma unroll
  for (int k = 0; k < kScatterItems; ++k) {
    int m = mi[k];
    if (m >= n_mats) m = -1;
    mi[k] = m;
    rk[k] = 0;
    const uint32_t active = __ballot_sync(0xffffffffu, m >= 0);
    if (m >= 0) {
      const uint32_t peers = __match_any_sync(active, m);
      const int leader = __ffs(peers) - 1;
      int32_t r0 = 0;
      if ((int)(threadIdx.x & 31) == leader) r0 = atomicAdd(&cnt[m], __popc(peers));
      r0 = __shfl_sync(peers, r0, leader);
      rk[k] = r0 + __popc(peers & lanemask_lt());
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // chunk-local segment offsets
    int32_t acc = 0;
    for (int m = 0; m < n_mats; ++m) {
      loc[m] = acc;
      acc += cnt[m];
    }
    loc[n_mats] = acc;
  }
  for (int i = threadIdx.x; i < n_mats; i += blockDim.x)
    base[i] = off[i] + (cnt[i] ? atomicAdd(cursor + i, cnt[i]) : 0);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScatterItems; ++k)
    if (mi[k] >= 0) S.src[loc[mi[k]] + rk[k]] = k * 256 + threadIdx.x;
  __syncthreads();
  // write each segment range contiguously: position p -> slot base[m] + p - loc[m]
  const int tot = loc[n_mats];
  auto slot_of = [&](int p) {
    int m = 0;
    while (p >= loc[m + 1]) ++m;  // n_mats <= 64, typically a handful
    return (int64_t)base[m] + (p - loc[m]);
  };
  if (gather) {
    for (int p = threadIdx.x; p < tot; p += blockDim.x) order[slot_of(p)] = (int32_t)(c0 + S.src[p]);
    return;
  }
  const float lod0 = lod_stride ? 0.f : __ldg(lod);
  for (int p = threadIdx.x; p < tot; p += blockDim.x) {
    const int64_t sl = slot_of(p);
    const int r = S.src[p];
    order[sl] = (int32_t)(c0 + r);
    p_lod[sl] = lod_stride ? S.lod[r] : lod0;
    p_urr[sl] = S.urr[r];
    reinterpret_cast<float2*>(p_uv)[sl] = make_float2(S.uv[2 * r], S.uv[2 * r + 1]);
#pragma unroll
    for (int j = 0; j < 3; ++j) p_wi[3 * sl + j] = S.wi[3 * r + j];
    if (wo) {
#pragma unroll
      for (int j = 0; j < 3; ++j) p_wo[3 * sl + j] = S.wo[3 * r + j];
    }
    if (u3) {
#pragma unroll
      for (int j = 0; j < 3; ++j) p_u3[3 * sl + j] = S.u3[3 * r + j];
    }
  }
}

int num_sms_multi() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

// Side streams for concurrent segment launches (per device, created once).
constexpr int kMaxSide = 32;
struct SideStreams {
  std::mutex mu;  // one fork..join enqueue at a time (the events are shared)
  cudaStream_t st[kMaxSide] = {};
  cudaEvent_t ev[kMaxSide + 1] = {};
  bool ready = false;
};
SideStreams g_side[16];

SideStreams& sides() {
  int dev = 0;
  cudaGetDevice(&dev);
  SideStreams& S = g_side[dev & 15];
  static std::mutex init_mu;
  std::lock_guard<std::mutex> g(init_mu);
  if (!S.ready) {
    for (int i = 0; i < kMaxSide; ++i) {
      cudaStreamCreateWithFlags(&S.st[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&S.ev[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&S.ev[kMaxSide], cudaEventDisableTiming);
    S.ready = true;
  }
  return S;
}
cudaStream_t side_stream(int m) { return sides().st[m % kMaxSide]; }
void fork_streams(cudaStream_t s, int k) {
  SideStreams& S = sides();
  cudaEventRecord(S.ev[kMaxSide], s);
  for (int i = 0; i < k && i < kMaxSide; ++i) cudaStreamWaitEvent(S.st[i], S.ev[kMaxSide], 0);
}
cudaError_t join_streams(cudaStream_t s, int k) {
  SideStreams& S = sides();
  for (int i = 0; i < k && i < kMaxSide; ++i) {
    cudaEventRecord(S.ev[i], S.st[i]);
    cudaStreamWaitEvent(s, S.ev[i], 0);
  }
  return cudaGetLastError();
}

int grid256(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

size_t multi_workspace_bytes(int64_t n, int32_t n_mats) {
  // counts, offsets(+1), cursor, bad flag | order | uv lod urr wi wo u3
  // (segments padded to 4 rows: n + 4 n_mats rows)
  const size_t rows = (size_t)n + 4 * (size_t)n_mats;
  // + 256-byte alignment of each of the 9 regions
  return 4096 + (size_t)(5 * n_mats + 3) * 4 + rows * (4 + 40 + 12);
}

struct MultiWs {
  int32_t *counts, *offsets, *cursor, *bad, *seg, *order;
  float *uv, *lod, *urr, *wi, *wo, *u3;
};

static MultiWs carve(void* ws, int64_t n_rows, int32_t n_mats) {
  const int64_t n = n_rows + 4 * (int64_t)n_mats;
  auto align = [](uintptr_t p) { return (p + 255) & ~(uintptr_t)255; };
  uintptr_t p = align((uintptr_t)ws);
  MultiWs w;
  w.counts = (int32_t*)p; p += n_mats * 4;
  w.offsets = (int32_t*)p; p += (n_mats + 1) * 4;
  w.cursor = (int32_t*)p; p += n_mats * 4;
  w.bad = (int32_t*)p; p += 4;
  p = align(p); w.seg = (int32_t*)p; p += 2 * n_mats * 4;
  p = align(p); w.order = (int32_t*)p; p += n * 4;
  p = align(p); w.uv = (float*)p; p += n * 8;
  p = align(p); w.lod = (float*)p; p += n * 4;
  p = align(p); w.urr = (float*)p; p += n * 4;
  p = align(p); w.wi = (float*)p; p += n * 12;
  p = align(p); w.wo = (float*)p; p += n * 12;
  p = align(p); w.u3 = (float*)p;
  return w;
}

// Per-segment launch arguments: the permuted inputs at row offset `off`,
// outputs straight to query order through `order` (mode-dependent outputs).
// Segments read the caller's arrays through the row order (gather, default)
// or a permuted copy made by the scatter (NMQ_MULTI_GATHER=0).
bool multi_gather() {
  static const bool g = [] {
    const char* e = getenv("NMQ_MULTI_GATHER");
    return !(e && e[0] == '0');
  }();
  return g;
}

static QueryArgs segment_args(const QueryArgs& a, const MultiWs& w, int64_t off) {
  QueryArgs sa{};
  if (multi_gather()) {
    sa = a;
    sa.idx = w.order + off;
    sa.out_idx = w.order + off;
    sa.seg = nullptr;
    sa.max_ctas = 0;
    return sa;
  }
  sa.uv = w.uv + 2 * off;
  sa.lod = w.lod + off;
  sa.lod_stride = 1;
  sa.u_rr = w.urr + off;
  sa.wi = w.wi + 3 * off;
  sa.wo = a.wo ? w.wo + 3 * off : nullptr;
  sa.u3 = a.u3 ? w.u3 + 3 * off : nullptr;
  sa.rgb = a.rgb;
  sa.albedo = a.albedo;
  sa.ws = a.ws;
  sa.pdf = a.pdf;
  sa.params9 = a.params9;
  sa.level = a.level;
  sa.out_idx = w.order + off;
  return sa;
}

// BINNED eval / sample+pdf / query (mode).  checked: `host_counts` / `bad` come back to the host (one
// D2H sync per call) so out-of-range ids are reported, empty segments are
// skipped and the others run concurrently on SM shares proportional to
// their sizes.  !checked: no host round trip — every segment launch reads its
// {base, count} from the device (QueryArgs::seg); ids out of range are
// dropped (their rows are left untouched).
cudaError_t multi_binned(const MatParams* const* mps, int32_t n_mats, int mode, const QueryArgs& a,
                         const int32_t* mat_id, void* ws, int32_t* host_counts, int32_t* bad,
                         bool checked, cudaStream_t s) {
  if (n_mats > kMaxMats) return cudaErrorInvalidValue;
  MultiWs w = carve(ws, a.n, n_mats);
  cudaError_t e;
  if ((e = cudaMemsetAsync(w.counts, 0, (3 * n_mats + 2) * 4, s)) != cudaSuccess) return e;
  {
    const int nb = grid256(a.n), cap = 4 * num_sms_multi();
    bin_count_kernel<<<nb < cap ? nb : cap, 256, 0, s>>>(a.n, n_mats, mat_id, w.counts, w.bad);
  }
  const bool gather = multi_gather();
  const size_t sm_bytes = scatter_smem_bytes(gather, a.lod_stride != 0, a.wo != nullptr, a.u3 != nullptr);
  if (max_dynamic_smem((const void*)bin_scatter_kernel) < (int)sm_bytes) return cudaErrorInvalidValue;
  bin_scatter_kernel<<<(unsigned)((a.n + kScatterRows - 1) / kScatterRows), 256, sm_bytes, s>>>(
      a.n, n_mats, mat_id, w.counts, w.seg, w.cursor, w.order, a.uv, a.lod, a.lod_stride, a.u_rr, a.wi,
      a.wo, a.u3, gather ? nullptr : w.uv, w.lod, w.urr, w.wi, w.wo, w.u3);
  g_launches += 2;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (!checked) {
    // one launch per material on its own stream, each on ~1/n_mats of the
    // SMs, so the segments run side by side (no serialized pipeline
    // fill/drain); forked from and joined back into `s` with events.  (The
    // host does not know the segment sizes here; full-grid launches that
    // keep a device-computed share of their CTAs measured slower — 9.5 vs
    // 12.8 G q/s on C4 — since surplus CTAs of one launch hold up the
    // dispatch of the next.)
    const int nsm = num_sms_multi();
    const int per = nsm / n_mats > 0 ? nsm / n_mats : 1;
    std::lock_guard<std::mutex> lock(sides().mu);
    fork_streams(s, n_mats);
    for (int m = 0; m < n_mats; ++m) {
      QueryArgs sa = segment_args(a, w, 0);
      sa.n = a.n;  // capacity bound; the segment's rows come from w.seg
      sa.seg = w.seg + 2 * m;
      sa.max_ctas = per;
      if ((e = launch_fused(*mps[m], mode, sa, side_stream(m))) != cudaSuccess) return e;
    }
    return join_streams(s, n_mats);
  }
  if ((e = cudaMemcpyAsync(host_counts, w.counts, n_mats * 4, cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return e;
  if ((e = cudaMemcpyAsync(bad, w.bad, 4, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if (*bad) return cudaErrorInvalidValue;
  // the counts are known here: the non-empty segments run side by side, each
  // on a share of the SMs proportional to its size (a coherent batch keeps
  // the whole GPU, a uniform mix splits it evenly)
  int64_t total = 0;
  for (int m = 0; m < n_mats; ++m) total += host_counts[m];
  const int nsm = num_sms_multi();
  std::lock_guard<std::mutex> lock(sides().mu);
  fork_streams(s, n_mats);
  int64_t off = 0;
  for (int m = 0; m < n_mats; ++m) {
    const int64_t c = host_counts[m];
    if (c > 0) {
      QueryArgs sa = segment_args(a, w, off);  // results go straight back to query order
      sa.n = c;
      const int64_t share = (int64_t)nsm * c / total;
      sa.max_ctas = share >= 1 ? (int32_t)share : 1;
      if ((e = launch_fused(*mps[m], mode, sa, side_stream(m))) != cudaSuccess) return e;
    }
    off += (c + 3) & ~3;
  }
  return join_streams(s, n_mats);
}

}  // namespace nmq
