// gs_engine.cu — host orchestration of the GridShift engine and its C-ABI (gridshift_c.h).
//
// One gs_run clusters every frame of the input.  Phases:
//   n-scale   K1 bounds -> K2 binning -> sort occupied cells -> K3 lex cell list
//   m-scale   per iteration: K4 neighbour lists + dataflow sweep, K5 rehome + stable sort +
//             ordered merge fold + index update + has_converged + root composition
//   n-scale   K7 label propagation, centroids out
// Frames are independent: they share one launch sequence, and a frame that has
// terminated is frozen (its cells are neither swept nor rehomed) while others keep iterating.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <climits>
#include <functional>
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gridshift_c.h"
#include "gs_kernels.cuh"
#include "gs_global.cuh"
#include "gs_resident.cuh"
#include "gs_mspp.cuh"

namespace {

constexpr int64_t kMaxDenseCells = int64_t(1) << 28;  // dense grid cap (u32 keys, <= ~10 GB)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool owned = true;  // false: a view into another allocation (the control block)
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p && owned) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void view(void* q, size_t n) {
    release();
    p = q;
    bytes = n;
    owned = false;
  }
};

int64_t ipow3(int d) {
  int64_t k = 1;
  for (int i = 0; i < d; ++i) k *= 3;
  return k;
}

unsigned blocks_for(int64_t n, int threads, int64_t cap = 1 << 20) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// Diagnostics and schedule overrides read from the environment exist only in debug builds
// (-DGS_DEBUG_KNOBS); the product library reads no environment variables.
const char* knob(const char* name) {
#ifdef GS_DEBUG_KNOBS
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// Kernel attributes (dynamic shared memory above 48 KB, non-portable cluster sizes) are per
// device: each launcher keeps a bitmask of the devices it has configured, set under a lock so a
// concurrent context (gs_tune's worker threads) never launches before the attribute is in.
std::mutex g_attr_mu;

template <typename K>
cudaError_t attr_once(std::atomic<uint64_t>& mask, int dev, K* kernel, int smem,
                      bool nonportable_cluster = false, bool* cluster_ok = nullptr) {
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (nonportable_cluster) {
    const bool ok = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                         1) == cudaSuccess;
    cudaGetLastError();
    if (cluster_ok) *cluster_ok = ok;
  }
  mask.fetch_or(bit, std::memory_order_release);
  return cudaSuccess;
}

}  // namespace

struct gs_ctx {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  uint32_t epoch = 0;

  // dense cell grid (clean invariant between runs: cnt = 0, qs = 0, idx = -1)
  DevBuf cnt, qs, idx, lab;
  int64_t dense_cap = 0;
  int qs_dim = 0;
  // per point
  DevBuf pts, slot, labels;
  // per cell (double-buffered state)
  DevBuf occ, occ_sorted, ckey[2], ccnt[2], S[2], S1, nbl, nbn, nbe, den, flag, nkey, vals,
      skey, sval, head, sid, segstart, parent, root, initkey, erec, lprod, rden, lvl, lsucc,
      order;
  int64_t cell_cap = 0, nbl_cap = 0;
  // per frame
  DevBuf fdone, fchanged, fadj, fm, fdisp, ffirst, fcount, ifirst, icount, fiters, fconv, fk,
      hist;
  int64_t frame_cap = 0;
  // misc
  DevBuf counters, errflag, bpart, cub_tmp, dbg, modes, tiles, dbox, epoch_dev;
  // control block: one allocation, one memset and one readback copy per run
  //   [errflag 32 B][counters 64 B][modes 96 B][fswept i64 x nf][fdone][fiters][fconv][fk][fout]
  //   (zeroed up to fk; read back whole)
  DevBuf ctl, fswept, fout;
  int64_t ctl_nf = 0;
  // bumped whenever a device buffer is (re)allocated: a cached graph holds raw pointers
  uint64_t alloc_gen = 0;
  int img_w = 0;  // GS_U8 rgbxy: image width of the current call
  int bin_rep_log2 = 0;  // K2 table replicas per cell (2^x): batched frames use 4
  const void* host_src = nullptr;  // pinned caller points read by K1 directly (zero copy)
  // multi-GPU shard state (gs_shard_*): the global key box from gs_shard_bin, and for
  // gs_shard_run the merged partial cells the run starts from instead of binning
  bool shard_box = false;
  bool shard_front = false;
  int64_t shard_m = 0;
  const uint32_t* shard_keys = nullptr;
  const uint32_t* shard_counts = nullptr;
  const int64_t* shard_sums = nullptr;
  DevBuf xsum, pkeys, pcounts, psums, npend;
  // component sweep of the global path (gs_global.cuh k_cc_* / k_sweep_comp)
  DevBuf ccpar, ccsize, cccur, ccoff, ccmem, ccloc, ccdesc, ccctr, ccgs;
  bool comp_ok = true;  // the component sweep can be launched on this device
  // MS++ all-SM loop (first grids beyond one CTA): particles, their keys, initial-cell roots
  DevBuf mpos, mpc, mkey, mroot, msnew;
  // pinned, device-mapped readback area: K7 stores the control block there (zero copy)
  void* pin = nullptr;
  void* pin_dev = nullptr;
  size_t pin_bytes = 0;
  // global path: small pinned area for the per-iteration readbacks (plan, packed frame state)
  void* hpin = nullptr;
  size_t hpin_bytes = 0;
  cudaEvent_t ev_plan = nullptr;
  DevBuf iterpack;  // device side of the packed end-of-iteration readback
  // the control block's zero region is zero (K7 re-zeroes it at the end of every run; any
  // other user of the block, or a run that stopped early, clears this and a memset follows)
  bool ctl_clean = false;
  // shape cache: a run whose frames all went straight to K8 lets later runs of the same
  // shape launch K8 optimistically (no host round trip between binning and labels)
  struct ShapeKey {
    int64_t n = 0, nf = 0;
    int d = 0, dtype = 0;
    double h = 0;
    int max_iter = 0;
    int img_w = 0;
    bool operator==(const ShapeKey& o) const {
      return n == o.n && nf == o.nf && d == o.d && dtype == o.dtype && h == o.h &&
             max_iter == o.max_iter && img_w == o.img_w;
    }
  } shape;
  int shape_ms = 0;
  GsBox shape_box{};
  int64_t shape_vol_frame = 0;
  // a few recent shapes (a whole-batch call and the frame groups of a host batch alternate)
  struct ShapeEntry {
    ShapeKey key;
    int ms = 0;
    GsBox box{};
    int64_t vol_frame = 0;
    uint64_t used = 0;
  };
  ShapeEntry shapes[4];
  uint64_t shape_tick = 0;
  // CUDA graph of the optimistic run for one (shape, caller buffers) combination
  struct GraphKey {
    ShapeKey shape;
    const void* points = nullptr;
    const void* labels = nullptr;
    uint32_t flags = 0;
    int on_device = 0;
    uint64_t gen = 0;
    uint64_t pbox_gen = 0;  // the predicted box baked into the graph (~0: bounds pass)
    bool operator==(const GraphKey& o) const {
      return shape == o.shape && points == o.points && labels == o.labels && flags == o.flags &&
             on_device == o.on_device && gen == o.gen && pbox_gen == o.pbox_gen;
    }
  } gkey;
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launches = 0;
  bool use_graphs = true;
  // last run (host side)
  GsBox box{};
  int64_t nframes = 0;
  int cur = 0;  // which ckey/ccnt/S buffer holds the final cells
  int64_t k_total = 0;
  std::vector<int32_t> h_ffirst;
  std::vector<int64_t> h_k;
  std::vector<int32_t> h_iters, h_conv, h_done;
  std::vector<std::vector<int64_t>> hist_m;
  std::vector<std::vector<double>> hist_d;
  bool have_run = false;
  // frame-group pipeline (gs_run on host frames): the copy stream stages group g+1 while
  // group g runs; the per-frame centroids of the whole call are kept on the host
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_copy[2] = {};
  DevBuf stage[2];
  // labels of a frame group leave by DMA on their own stream while the next groups run
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t ev_d2h[2] = {};
  DevBuf lab_stage[2];
  bool grouped = false;
  int64_t group_f0 = 0;
  // predicted key box: the box of the last successful run of this (n, frames, d, dtype, h)
  // replaces the bounds pass (K2 flags any point outside it and the run is redone)
  bool pbox_valid = false;
  GsBox pbox{};
  int64_t pbox_n = 0, pbox_nf = 0;
  int pbox_d = 0, pbox_dtype = 0, pbox_w = 0;
  double pbox_h = 0;
  uint64_t pbox_gen = 0;
  int predicted = 0;      // this launch of K2 bins against the predicted box
  uint32_t sweep_flags = 0;  // GS_DEBUG_SWEEP_* of the current run
  // per-context sweep schedule (a cluster shape the device refused is not retried)
  bool flow_ok = true, cluster16_ok = true, cluster_ok = true;  // first frame of the last group (its slot/label state is live)
  std::vector<double> g_cent;
  std::vector<int64_t> g_cent_off;
  gs_stats stats{};
  bool stats_times_pending = false;
  unsigned ev_mask = 0;  // which phase events this run records
  cudaEvent_t ev[12] = {};
};

namespace {

#define GS_CK(call)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
      return (e_ == cudaErrorMemoryAllocation) ? GS_E_OOM : GS_E_CUDA;               \
    }                                                                                \
  } while (0)

#define GS_TRY(expr)             \
  do {                           \
    gs_status s_ = (expr);       \
    if (s_ != GS_OK) return s_;  \
  } while (0)

gs_status fail(gs_ctx* ctx, gs_status s, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return s;
}

gs_status grow(gs_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes <= b.bytes) return GS_OK;
  b.release();
  size_t want = std::max<size_t>(bytes, 256);
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    b.p = nullptr;
    cudaGetLastError();
    return fail(ctx, GS_E_OOM, "cudaMalloc(" + std::to_string(want) + ") failed");
  }
  b.bytes = want;
  b.owned = true;
  ++ctx->alloc_gen;
  return GS_OK;
}

// Phase events; recorded as external event nodes while the stream is being captured so the
// graph replay records them too (elapsed times keep working on the graph path).
// Events cost ~3.5 us each as graph nodes (measured: 8 events = 28 us of a 170 us cfg2 run),
// so they are recorded only when the caller asks: GS_TIME_KERNEL (the binning kernel's pair,
// 6/7) or GS_TIME_PHASES (all).
gs_status rec_event(gs_ctx* ctx, int i) {
  if (!((ctx->ev_mask >> i) & 1u)) return GS_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  GS_CK(cudaStreamIsCapturing(ctx->stream, &cs));
  GS_CK(cudaEventRecordWithFlags(ctx->ev[i], ctx->stream,
                                 cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal
                                                                     : cudaEventRecordDefault));
  return GS_OK;
}

gs_status check_launch(gs_ctx* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, GS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  ctx->stats.kernel_launches++;
  return GS_OK;
}

#define GS_LAUNCHED(name) GS_TRY(check_launch(ctx, name))

gs_status check_lib(gs_ctx* ctx, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, GS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  ctx->stats.lib_calls++;
  return GS_OK;
}

gs_status validate(const gs_input* in, const gs_config* cfg) {
  if (!in || !cfg) return GS_E_INVALID_PARAMETER;
  if (!(cfg->h > 0.0) || !std::isfinite(cfg->h)) return GS_E_INVALID_BANDWIDTH;
  if (in->n < 1 || in->batch < 1) return in->n < 1 ? GS_E_EMPTY_INPUT : GS_E_INVALID_PARAMETER;
  if (in->d < 1 || in->d > GS_MAX_DIM) return GS_E_INVALID_PARAMETER;
  if (in->dtype != GS_F32 && in->dtype != GS_F64 && in->dtype != GS_U8)
    return GS_E_INVALID_PARAMETER;
  if (in->dtype == GS_U8) {  // pixels: rgb (d = 3) or rgbxy (d = 5, width in `reserved`)
    if (in->d != 3 && in->d != 5) return GS_E_INVALID_PARAMETER;
    if (in->d == 5 && (in->reserved < 2 || in->n % in->reserved != 0 || in->n / in->reserved < 2))
      return GS_E_INVALID_PARAMETER;
  }
  if (cfg->max_iter < 1) return GS_E_INVALID_PARAMETER;
  if (!in->points) return GS_E_INVALID_PARAMETER;
  if (in->n * in->batch > (int64_t(1) << 40)) return GS_E_INVALID_PARAMETER;
  return GS_OK;
}

// bytes of the raw point array of `in` (GS_U8: 3 bytes per pixel whatever d is)
size_t input_bytes(const gs_input* in) {
  const size_t per = in->dtype == GS_U8 ? 3 : (in->dtype == GS_F32 ? 4 : 8) * (size_t)in->d;
  return per * (size_t)in->n * (size_t)in->batch;
}

// Dense grid: grow to hold `cells` cells of dimension d; fresh memory gets the clean state.
gs_status ensure_dense(gs_ctx* ctx, int64_t cells, int d) {
  if (cells <= ctx->dense_cap && d <= ctx->qs_dim) return GS_OK;
  int64_t cap = std::max<int64_t>(cells, ctx->dense_cap);
  int qd = std::max(d, ctx->qs_dim);
  ctx->cnt.release();
  ctx->qs.release();
  ctx->idx.release();
  ctx->lab.release();
  ctx->dense_cap = 0;
  GS_TRY(grow(ctx, ctx->cnt, sizeof(uint32_t) * cap));
  GS_TRY(grow(ctx, ctx->qs, sizeof(unsigned long long) * cap * qd));
  GS_TRY(grow(ctx, ctx->idx, sizeof(int32_t) * cap));
  // (+65536: a u16 slot left by an aborted run can reach past the last frame; K7 reads it)
  GS_TRY(grow(ctx, ctx->lab, sizeof(int32_t) * (cap + 65536)));
  GS_CK(cudaMemsetAsync(ctx->cnt.p, 0, sizeof(uint32_t) * cap, ctx->stream));
  GS_CK(cudaMemsetAsync(ctx->qs.p, 0, sizeof(unsigned long long) * cap * qd, ctx->stream));
  GS_CK(cudaMemsetAsync(ctx->idx.p, 0xff, sizeof(int32_t) * cap, ctx->stream));
  ctx->dense_cap = cap;
  ctx->qs_dim = qd;
  return GS_OK;
}

gs_status ensure_cells(gs_ctx* ctx, int64_t m, int d) {
  if (m <= ctx->cell_cap) return GS_OK;
  int64_t c = std::max<int64_t>(m, 1024);
  for (DevBuf* b : {&ctx->occ, &ctx->occ_sorted, &ctx->ckey[0], &ctx->ckey[1], &ctx->ccnt[0],
                    &ctx->ccnt[1], &ctx->nkey, &ctx->vals, &ctx->skey, &ctx->sval})
    GS_TRY(grow(ctx, *b, sizeof(uint32_t) * c));
  for (DevBuf* b : {&ctx->nbn, &ctx->nbe, &ctx->head, &ctx->sid, &ctx->segstart, &ctx->parent,
                    &ctx->root, &ctx->initkey})
    GS_TRY(grow(ctx, *b, sizeof(int32_t) * c));
  GS_TRY(grow(ctx, ctx->den, sizeof(unsigned long long) * c));
  for (DevBuf* b : {&ctx->S[0], &ctx->S[1], &ctx->S1})
    GS_TRY(grow(ctx, *b, sizeof(double) * c * GS_MAX_DIM));
  if (ctx->flag.bytes < sizeof(uint32_t) * c) {
    GS_TRY(grow(ctx, ctx->flag, sizeof(uint32_t) * c));
    GS_CK(cudaMemsetAsync(ctx->flag.p, 0, ctx->flag.bytes, ctx->stream));
  }
  // CUB temporaries for the largest sort/scan on c items
  size_t t1 = 0, t2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (uint32_t*)nullptr, (int)c, 0, 32,
                                  ctx->stream);
  cub::DeviceScan::InclusiveSum(nullptr, t2, (int32_t*)nullptr, (int32_t*)nullptr, (int)c,
                                ctx->stream);
  size_t t3 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, t3, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)c, 0,
                                 32, ctx->stream);
  GS_TRY(grow(ctx, ctx->cub_tmp, std::max({t1, t2, t3})));
  ctx->cell_cap = c;
  return GS_OK;
}

// control-block geometry for nf frames
constexpr size_t kCtlHeader = 192;
size_t ctl_zero_bytes(int64_t nf) { return kCtlHeader + 8 * (size_t)nf + 12 * (size_t)nf; }
size_t ctl_bytes(int64_t nf) { return kCtlHeader + 8 * (size_t)nf + 20 * (size_t)nf; }

gs_status ensure_ctl(gs_ctx* ctx, int64_t nf) {
  if (nf <= ctx->ctl_nf && ctx->ctl.p) return GS_OK;
  for (DevBuf* b : {&ctx->errflag, &ctx->counters, &ctx->modes, &ctx->fswept, &ctx->fdone,
                    &ctx->fiters, &ctx->fconv, &ctx->fk, &ctx->fout})
    b->release();
  ctx->ctl.release();
  GS_TRY(grow(ctx, ctx->ctl, ctl_bytes(nf)));
  GS_CK(cudaMemsetAsync(ctx->ctl.p, 0, ctl_bytes(nf), ctx->stream));
  ctx->ctl_clean = true;
  char* p = ctx->ctl.as<char>();
  ctx->errflag.view(p, 32);
  ctx->counters.view(p + 32, 64);
  ctx->modes.view(p + 96, 96);
  p += kCtlHeader;
  ctx->fswept.view(p, 8 * nf);  p += 8 * nf;
  ctx->fdone.view(p, 4 * nf);   p += 4 * nf;
  ctx->fiters.view(p, 4 * nf);  p += 4 * nf;
  ctx->fconv.view(p, 4 * nf);   p += 4 * nf;
  ctx->fk.view(p, 4 * nf);      p += 4 * nf;
  ctx->fout.view(p, 4 * nf);
  ctx->ctl_nf = nf;
  return GS_OK;
}

gs_status ensure_frames(gs_ctx* ctx, int64_t nf) {
  GS_TRY(ensure_ctl(ctx, nf));
  if (nf <= ctx->frame_cap) return GS_OK;
  for (DevBuf* b : {&ctx->fchanged, &ctx->fadj, &ctx->fm, &ctx->ffirst, &ctx->fcount})
    GS_TRY(grow(ctx, *b, sizeof(int32_t) * nf));
  GS_TRY(grow(ctx, ctx->ifirst, sizeof(int32_t) * (nf + 1)));  // [nf] = m0
  GS_TRY(grow(ctx, ctx->fdisp, sizeof(unsigned long long) * nf));
  ctx->frame_cap = nf;
  return GS_OK;
}

int bits_for(int64_t v) {  // bits needed to represent values < v
  int b = 1;
  while (b < 32 && (int64_t(1) << b) < v) ++b;
  return b;
}

// Box from per-dim data min/max (host).  floor(min/h) <= floor(x/h) <= floor(max/h) for every
// x by monotonicity of IEEE division and floor.
gs_status make_box(gs_ctx* ctx, int d, double h, int64_t n, int64_t nframes, const double* mn,
                   const double* mx, GsBox* b) {
  std::memset(b, 0, sizeof(*b));
  b->d = d;
  b->h = h;
  b->inv_h = 1.0 / h;
  b->F = gs_fixed_shift(n, h);
  b->scale = std::ldexp(1.0, b->F);
  b->inv_scale = std::ldexp(1.0, -b->F);
  b->n = n;
  b->nframes = nframes;
  double vol = 1.0;
  for (int c = 0; c < d; ++c) {
    double lo = std::floor(mn[c] / h), hi = std::floor(mx[c] / h);
    if (!(std::fabs(lo) < 4e15) || !(std::fabs(hi) < 4e15))
      return fail(ctx, GS_E_KEY_RANGE, "cell keys exceed the int64 key range");
    b->kmin[c] = (int64_t)lo - GS_APRON;
    b->ext[c] = (int64_t)hi - (int64_t)lo + 1 + 2 * GS_APRON;
    vol *= (double)b->ext[c];
  }
  if (vol * (double)nframes > (double)kMaxDenseCells)
    return fail(ctx, GS_E_KEY_RANGE,
                "key box of " + std::to_string((long long)(vol * nframes)) +
                    " cells exceeds the dense cell grid (2^28)");
  int64_t s = 1;
  for (int c = d - 1; c >= 0; --c) {
    b->stride[c] = s;
    s *= b->ext[c];
  }
  b->vol_frame = s;
  b->vol_total = s * nframes;
  return GS_OK;
}

// Box for an injected cell state (test hook): covers the keys and floor(centroid/h).
gs_status make_box_from_cells(gs_ctx* ctx, int d, double h, int64_t m, const int64_t* keys,
                              const double* cent, GsBox* b) {
  std::vector<double> mn(d, INFINITY), mx(d, -INFINITY);
  for (int64_t i = 0; i < m; ++i)
    for (int c = 0; c < d; ++c) {
      double kh = (double)keys[i * d + c] * h;  // any x with floor(x/h) == key
      double lo = std::min(cent[i * d + c], kh), hi = std::max(cent[i * d + c], kh);
      mn[c] = std::min(mn[c], lo);
      mx[c] = std::max(mx[c], hi);
    }
  GS_TRY(make_box(ctx, d, h, 1 << 20, 1, mn.data(), mx.data(), b));
  for (int64_t i = 0; i < m; ++i)
    for (int c = 0; c < d; ++c) {
      int64_t rel = keys[i * d + c] - b->kmin[c];
      if (rel < GS_APRON || rel >= b->ext[c] - GS_APRON) {  // widen: keys define the box
        int64_t lo = std::min<int64_t>(keys[i * d + c], b->kmin[c] + GS_APRON);
        int64_t hi = std::max<int64_t>(keys[i * d + c], b->kmin[c] + b->ext[c] - GS_APRON - 1);
        b->kmin[c] = lo - GS_APRON;
        b->ext[c] = hi - lo + 1 + 2 * GS_APRON;
      }
    }
  int64_t s = 1;
  for (int c = d - 1; c >= 0; --c) {
    b->stride[c] = s;
    s *= b->ext[c];
  }
  b->vol_frame = s;
  b->vol_total = s;
  if (s > kMaxDenseCells) return fail(ctx, GS_E_KEY_RANGE, "injected key box too large");
  return GS_OK;
}

template <int D, typename T>
gs_status launch_bounds_bin_t(gs_ctx* ctx, const void* pts, int64_t ntot, bool bounds,
                              unsigned nblk, double h, int64_t n, int64_t nf) {
  const int img_w = ctx->img_w;
  if (bounds) {
    unsigned* ctr = ctx->counters.as<unsigned>();
    int* err = ctx->errflag.as<int>();
    const int F = gs_fixed_shift(n, h);
    // zero copy: read the caller's pinned points, store the device copy K2 reads
    const void* src = ctx->host_src ? ctx->host_src : pts;
    T* copy = ctx->host_src ? (T*)pts : nullptr;
    gs::k_bounds_box<D, T><<<nblk, 256, 0, ctx->stream>>>(
        (const T*)src, ntot, ctx->bpart.as<double>(), h, F, n, nf, ctx->dense_cap,
        ctx->dbox.as<GsBox>(), err, (long long*)(err + 2), ctr + 6,
        ctx->epoch_dev.as<unsigned>(), img_w, copy);
    GS_LAUNCHED("k_bounds_box");
  } else {
    // privatised binning: one 1024-thread CTA per SM at most, >= 1024 points per CTA; the
    // geometry comes from the host copy of the key box (ctx->box) as kernel parameters
    const unsigned grid = blocks_for(ntot, 1024, (int64_t)ctx->num_sms * gs::kBinCtas);
    static std::atomic<uint64_t> done{0};
    GS_CK(attr_once(done, ctx->device, gs::k_bin<D, T>, gs::kBinSmemBytes));
    const gs::BinParams P = gs::make_bin_params<D>(ctx->box, 4, ctx->bin_rep_log2, ctx->predicted);
    gs::k_bin<D, T><<<grid, gs::kBinThreads, gs::kBinSmemBytes, ctx->stream>>>(
        (const T*)pts, ntot, P, ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>(),
        ctx->slot.p, ctx->errflag.as<int>(), img_w,
        ctx->predicted ? ctx->dbox.as<GsBox>() : nullptr,
        ctx->predicted ? ctx->epoch_dev.as<unsigned>() : nullptr, ctx->box);
    GS_LAUNCHED("k_bin");
  }
  return GS_OK;
}

template <int D>
gs_status launch_bounds_bin(gs_ctx* ctx, const void* pts, int dtype, int64_t ntot, bool bounds,
                            unsigned nblk, double h = 0, int64_t n = 0, int64_t nf = 0) {
  if (dtype == GS_F32) return launch_bounds_bin_t<D, float>(ctx, pts, ntot, bounds, nblk, h, n, nf);
  if (dtype == GS_F64) return launch_bounds_bin_t<D, double>(ctx, pts, ntot, bounds, nblk, h, n, nf);
  if constexpr (D == 3 || D == 5)  // GS_U8 pixels: rgb / rgbxy
    return launch_bounds_bin_t<D, uint8_t>(ctx, pts, ntot, bounds, nblk, h, n, nf);
  return fail(ctx, GS_E_INVALID_PARAMETER, "8-bit pixels need d = 3 or 5");
}

gs_status dispatch_bounds_bin(gs_ctx* ctx, const void* pts, int dtype, int d, int64_t ntot,
                              bool bounds, unsigned nblk, double h = 0, int64_t n = 0,
                              int64_t nf = 0) {
  switch (d) {
#define GS_CASE(D) \
  case D:          \
    return launch_bounds_bin<D>(ctx, pts, dtype, ntot, bounds, nblk, h, n, nf);
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
    GS_CASE(7) GS_CASE(8) GS_CASE(9) GS_CASE(10) GS_CASE(11) GS_CASE(12)
#undef GS_CASE
  }
  return fail(ctx, GS_E_INVALID_PARAMETER, "d out of range");
}

gs_status read_err(gs_ctx* ctx, int* out) {
  GS_CK(cudaMemcpyAsync(out, ctx->errflag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaStreamSynchronize(ctx->stream));
  return GS_OK;
}

// device scratch layout
//   errflag (int[8]): [0] error bits, [2..3] int64 cells needed when bit 32 is set
//   counters (unsigned[16]): [0] m0, [1] global-sweep ticket, [2] largest frame (cells),
//                            [4] K8 deferred
constexpr int64_t kDefaultDenseCells = int64_t(1) << 22;

// The device found a key box larger than the allocated grid: grow to it, or refuse loudly
// when it exceeds the dense-grid cap (no silent approximation).
gs_status grow_dense_for(gs_ctx* ctx, long long need, int d) {
  if (need <= 0 || need > kMaxDenseCells)
    return fail(ctx, GS_E_KEY_RANGE,
                "key box of " + std::to_string(need) + " cells exceeds the dense cell grid (2^28)");
  return ensure_dense(ctx, (int64_t)need, d);
}

// The control block's zero region must be zero when a run starts; K7 leaves it so.  Outside
// a graph capture a dirty block is cleared here; a captured run relies on the invariant (the
// caller clears before launching the graph).
gs_status clean_ctl(gs_ctx* ctx) {
  if (ctx->ctl_clean) return GS_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  GS_CK(cudaStreamIsCapturing(ctx->stream, &cs));
  if (cs == cudaStreamCaptureStatusActive) return GS_OK;
  GS_CK(cudaMemsetAsync(ctx->ctl.p, 0, ctl_zero_bytes(ctx->ctl_nf), ctx->stream));
  ctx->ctl_clean = true;
  return GS_OK;
}

// n-scale phase with no host round trip: control block cleared -> bounds + device box ->
// privatised binning -> single-pass compaction (cells come out lexicographically sorted, with
// per-frame first indices).  Errors (non-finite input, key box beyond the grid) surface in
// errflag at the next sync.  vol_hint sizes the compaction grid (any value is correct).
gs_status launch_nscale(gs_ctx* ctx, const void* dpts, int dtype, int d, int64_t n, int64_t nf,
                        double h, int64_t vol_hint = 0, const GsBox* pbox = nullptr) {
  cudaStream_t st = ctx->stream;
  const int64_t ntot = n * nf;
  const unsigned nblk = blocks_for(ntot, 256 * 4, (int64_t)ctx->num_sms * 4);
  // batched frames (images): few distinct cells per warp -> 4 lane-chosen replicas per cell
  // in K2's table (GS_BIN_REPLICAS overrides: 0, 1 or 2 = log2 of the replica count)
  {
    const char* v = knob("GS_BIN_REPLICAS");
    ctx->bin_rep_log2 = v ? std::max(0, std::min(2, atoi(v))) : (nf > 1 ? 2 : 0);
  }
  GS_TRY(grow(ctx, ctx->bpart, sizeof(double) * nblk * d * 2));
  GS_TRY(grow(ctx, ctx->dbox, sizeof(GsBox)));
  GS_TRY(ensure_dense(ctx, std::max<int64_t>(ctx->dense_cap, kDefaultDenseCells), d));
  GS_TRY(ensure_cells(ctx, std::min<int64_t>(ntot, ctx->dense_cap), d));
  GS_TRY(ensure_frames(ctx, nf));
  GS_TRY(grow(ctx, ctx->slot, sizeof(uint32_t) * ntot));
  const int64_t ntiles = ctx->dense_cap / gs::kOccTile + 1;
  if (ctx->tiles.bytes < sizeof(unsigned long long) * ntiles) {  // epoch-tagged: cleared once
    GS_TRY(grow(ctx, ctx->tiles, sizeof(unsigned long long) * ntiles));
    GS_CK(cudaMemsetAsync(ctx->tiles.p, 0, ctx->tiles.bytes, st));
  }
  if (!ctx->epoch_dev.p) {
    GS_TRY(grow(ctx, ctx->epoch_dev, 16));
    GS_CK(cudaMemsetAsync(ctx->epoch_dev.p, 0, 16, st));
  }
  GS_TRY(clean_ctl(ctx));
  ctx->ctl_clean = false;  // until K7 of this run re-zeroes it
  if (pbox) {  // the predicted box: no bounds pass (K2 checks every point against it)
    if (ctx->host_src)  // zero-copy pinned input: K1 is the copy (its box is not used)
      GS_TRY(dispatch_bounds_bin(ctx, dpts, dtype, d, ntot, true, nblk, h, n, nf));
    ctx->box = *pbox;  // K2's block 0 stores it as the device box and bumps the run epoch
  } else {
    // bounds pass, then the box to the host: K2's geometry is kernel parameters
    GS_TRY(dispatch_bounds_bin(ctx, dpts, dtype, d, ntot, true, nblk, h, n, nf));
    int hdr[8];
    GS_CK(cudaMemcpyAsync(hdr, ctx->errflag.p, 32, cudaMemcpyDeviceToHost, st));
    GS_CK(cudaMemcpyAsync(&ctx->box, ctx->dbox.p, sizeof(GsBox), cudaMemcpyDeviceToHost, st));
    GS_CK(cudaStreamSynchronize(st));
    if (hdr[0] & GS_ERR_SKIP) return GS_OK;  // the caller reads the error bits
  }
  ctx->predicted = pbox ? 1 : 0;
  GS_TRY(rec_event(ctx, 6));
  const gs_status sb = dispatch_bounds_bin(ctx, dpts, dtype, d, ntot, false, nblk);
  ctx->predicted = 0;
  GS_TRY(sb);
  GS_TRY(rec_event(ctx, 7));
  unsigned* cnt32 = ctx->counters.as<unsigned>();
  const int64_t vt = vol_hint > 0 ? std::min(vol_hint, ctx->dense_cap) : ctx->dense_cap;
  const unsigned tg = (unsigned)std::min<int64_t>(vt / gs::kOccTile + 1, (int64_t)ctx->num_sms * 4);
  gs::k_occ<<<tg, 256, 0, st>>>(
      ctx->dbox.as<GsBox>(), ctx->epoch_dev.as<unsigned>(), ctx->tiles.as<unsigned long long>(),
      cnt32 + 5, cnt32, ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>(),
      ctx->ckey[0].as<uint32_t>(), ctx->ccnt[0].as<uint32_t>(), ctx->S[0].as<double>(),
      ctx->idx.as<int32_t>(), ctx->root.as<int32_t>(), ctx->initkey.as<uint32_t>(),
      ctx->ifirst.as<int32_t>(), ctx->errflag.as<int>());
  GS_LAUNCHED("k_occ");
  return GS_OK;
}

gs_status ensure_hpin(gs_ctx* ctx, size_t need) {
  if (need > ctx->hpin_bytes) {
    if (ctx->hpin) {
      GS_CK(cudaStreamSynchronize(ctx->stream));
      cudaFreeHost(ctx->hpin);
    }
    ctx->hpin = nullptr;
    ctx->hpin_bytes = 0;
    need = std::max<size_t>(need, 4096);
    GS_CK(cudaHostAlloc(&ctx->hpin, need, cudaHostAllocDefault));
    ctx->hpin_bytes = need;
  }
  if (!ctx->ev_plan) GS_CK(cudaEventCreateWithFlags(&ctx->ev_plan, cudaEventDisableTiming));
  return GS_OK;
}

template <int D>
gs_status launch_sweep_levels_d(gs_ctx* ctx, int64_t m, const int32_t* eoff,
                                const int32_t* loff) {
  // pending counts + queue in smem when they fit (8 bytes per cell), else in global scratch
  constexpr size_t kBudget = 220 * 1024;
  const size_t stage = (size_t)1024 * D * 8;
  const int smem_cells = (int)std::min<int64_t>(m, (int64_t)((kBudget - stage) / 8));
  if (knob("GS_DEBUG_KAHN")) {
    GS_TRY(grow(ctx, ctx->dbg, 64));
    GS_CK(cudaMemsetAsync(ctx->dbg.p, 0, 32, ctx->stream));
  }
  const size_t smem = stage + (size_t)smem_cells * 8;
  static std::atomic<uint64_t> done{0};
  GS_CK(attr_once(done, ctx->device, gs::k_sweep_kahn<D>, (int)kBudget));
  gs::k_sweep_kahn<D><<<1, 1024, smem, ctx->stream>>>(
      (int)m, smem_cells, ctx->nbn.as<int32_t>(), ctx->nbe.as<int32_t>(), eoff, loff,
      ctx->erec.as<unsigned long long>(), ctx->lprod.as<double>(), ctx->lsucc.as<int32_t>(),
      ctx->den.as<uint32_t>(), ctx->rden.as<double>(), ctx->S[ctx->cur].as<double>(),
      ctx->S1.as<double>(), ctx->lvl.as<int>(), ctx->order.as<int>(),
      knob("GS_DEBUG_KAHN") ? (long long*)ctx->dbg.p : nullptr);
  GS_LAUNCHED("k_sweep_kahn");
  if (knob("GS_DEBUG_KAHN")) {
    long long h[4];
    GS_CK(cudaMemcpyAsync(h, ctx->dbg.p, 32, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CK(cudaStreamSynchronize(ctx->stream));
    fprintf(stderr, "kahn m=%lld levels=%lld cells=%lld thread0_cycles=%lld\n", (long long)m, h[0], h[1], h[2]);
    GS_CK(cudaMemsetAsync(ctx->dbg.p, 0, 32, ctx->stream));
  }
  return GS_OK;
}

gs_status launch_sweep_levels(gs_ctx* ctx, int d, int64_t m, const int32_t* eoff,
                              const int32_t* loff) {
  switch (d) {
#define GS_CASE(D) \
  case D:          \
    return launch_sweep_levels_d<D>(ctx, m, eoff, loff);
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
    GS_CASE(7) GS_CASE(8) GS_CASE(9) GS_CASE(10) GS_CASE(11) GS_CASE(12)
#undef GS_CASE
  }
  return fail(ctx, GS_E_INVALID_PARAMETER, "d out of range");
}

// Global path, d <= 6: neighbour lists at a fixed stride, then the single-CTA Kahn sweep with
// the operand rows in L2 (gs_global.cuh).  Q = ctx->S1: rows [0, m) = S1 after the sweep.
// own_lo/own_hi/halo (multi-GPU slabs, gs_dist): cells outside [own_lo, own_hi) are the
// neighbouring slabs' boundary layers, frozen in the lists; `halo` writes their Q / P1 rows
// between the lists and the sweep
struct SweepHalo {
  int own_lo = 0, own_hi = INT_MAX;
  std::function<gs_status(double*)> rows;
};

template <int D>
gs_status launch_global_sweep_d(gs_ctx* ctx, int64_t m, int K, const SweepHalo* halo = nullptr) {
  if (halo) GS_TRY(grow(ctx, ctx->npend, 4 * (size_t)m));
  cudaStream_t st = ctx->stream;
  const GsBox& b = ctx->box;
  const int KP = (K + 3) & ~3;
  GS_TRY(grow(ctx, ctx->erec, 4 * (size_t)m * KP));  // the lists (u32 rows)
  GS_TRY(grow(ctx, ctx->rden, 8 * (size_t)m));
  GS_TRY(grow(ctx, ctx->S1, 8 * (size_t)(2 * m + 2) * D));
  GS_TRY(grow(ctx, ctx->lvl, 4 * (size_t)(m / 4 + 2)));  // pending counts (global fallback)
  GS_TRY(grow(ctx, ctx->order, 4 * (size_t)m));          // queue (global fallback)
  uint32_t* lists = ctx->erec.as<uint32_t>();
  double* Q = ctx->S1.as<double>();
  const int cur = ctx->cur;
  gs::k_nbr_lists<D><<<blocks_for(m, 256), 256, 0, st>>>(
      (int)m, b, K, KP, ctx->ckey[cur].as<uint32_t>(), ctx->ccnt[cur].as<uint32_t>(),
      ctx->S[cur].as<double>(), ctx->idx.as<int32_t>(), ctx->fdone.as<int32_t>(), lists,
      ctx->nbn.as<int32_t>(), ctx->nbe.as<int32_t>(), ctx->den.as<uint32_t>(),
      ctx->rden.as<double>(), Q, ctx->fm.as<int32_t>(), halo ? halo->own_lo : 0,
      halo ? halo->own_hi : INT_MAX, halo ? ctx->npend.as<int32_t>() : nullptr);
  const int32_t* pinit = halo ? ctx->npend.as<int32_t>() : nullptr;
  GS_LAUNCHED("k_nbr_lists");
  if (halo && halo->rows) GS_TRY(halo->rows(Q));
  const uint32_t dbg0 = ctx->sweep_flags;
  if constexpr (D <= 3) {
    // the component sweep (r2): connected components of the active cells swept independently,
    // one CTA each with everything in shared memory, when every component fits a CTA
    if (!halo && ctx->comp_ok &&
        !(dbg0 & (GS_DEBUG_SWEEP_FLOW | GS_DEBUG_SWEEP_LEVELS | GS_DEBUG_SWEEP_SINGLE)) &&
        m <= gs::kCcMaxCells) {
      for (DevBuf* bb : {&ctx->ccpar, &ctx->cccur, &ctx->ccoff, &ctx->ccmem})
        GS_TRY(grow(ctx, *bb, 4 * (size_t)m));
      GS_TRY(grow(ctx, ctx->ccloc, 4 * (size_t)m * D));   // box min corners (per root)
      GS_TRY(grow(ctx, ctx->ccsize, 4 * (size_t)m * D));  // box max corners (per root)
      GS_TRY(grow(ctx, ctx->ccgs, 4 * (size_t)m));        // component sizes (per root)
      GS_TRY(grow(ctx, ctx->ccdesc, 16 * (size_t)m));
      GS_TRY(grow(ctx, ctx->ccctr, 64));
      int32_t* root = ctx->ccpar.as<int32_t>();
      static std::atomic<uint64_t> done_s{0};
      const unsigned mb0 = blocks_for(m, 256);
      gs::k_cc_init<D><<<mb0, 256, 0, st>>>((int)m, KP, lists, ctx->nbe.as<int32_t>(), root,
                                            ctx->ccgs.as<int32_t>(), ctx->cccur.as<int32_t>(),
                                            ctx->ccloc.as<int32_t>(), ctx->ccsize.as<int32_t>());
      GS_LAUNCHED("k_cc_init");
      for (int jp = 0; jp < 2; ++jp) {
        gs::k_cc_jump<<<mb0, 256, 0, st>>>((int)m, root);
        GS_LAUNCHED("k_cc_jump");
      }
      gs::k_cc_hook<D><<<mb0, 256, 0, st>>>((int)m, KP, lists, ctx->nbe.as<int32_t>(), root);
      GS_LAUNCHED("k_cc_hook");
      gs::k_cc_count<D><<<mb0, 256, 0, st>>>((int)m, b, ctx->ckey[cur].as<uint32_t>(), root,
                                             ctx->ccgs.as<int32_t>(), ctx->ccloc.as<int32_t>(),
                                             ctx->ccsize.as<int32_t>());
      GS_LAUNCHED("k_cc_count");
      GS_CK(cudaMemsetAsync(ctx->ccctr.p, 0, 48, st));
      gs::k_cc_plan_par<D><<<mb0, 256, 0, st>>>(
          (int)m, ctx->ccgs.as<int32_t>(), ctx->ccloc.as<int32_t>(), ctx->ccsize.as<int32_t>(),
          ctx->ccoff.as<int32_t>(), ctx->ccdesc.as<int32_t>(),
          ctx->ccctr.as<unsigned long long>());
      GS_LAUNCHED("k_cc_plan");
      // The plan goes to the host while the sweep already runs: k_cc_scatter and k_sweep_comp
      // read it on the device (CTAs take components by ticket; a plan that does not fit a CTA
      // makes the launch a no-op), so the host's wait for it overlaps the sweep.
      constexpr size_t kCompBudget = 224 * 1024;
      GS_TRY(ensure_hpin(ctx, 64));
      long long* plan = (long long*)ctx->hpin;
      GS_CK(cudaMemcpyAsync(plan, ctx->ccctr.p, 24, cudaMemcpyDeviceToHost, st));
      GS_CK(cudaEventRecord(ctx->ev_plan, st));
      {
        const unsigned mb = blocks_for(m, 256);
        gs::k_cc_scatter<<<mb, 256, 0, st>>>((int)m, root, ctx->ccoff.as<int32_t>(),
                                             ctx->cccur.as<int32_t>(), ctx->ccmem.as<int32_t>());
        GS_LAUNCHED("k_cc_scatter");
        GS_CK(attr_once(done_s, ctx->device, gs::k_sweep_comp<D>, (int)kCompBudget));
        const unsigned cg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms, m / 2));
        gs::k_sweep_comp<D><<<cg, 256, kCompBudget, st>>>(
            (int)m, b, ctx->ccdesc.as<int32_t>(), ctx->ccmem.as<int32_t>(),
            ctx->ccloc.as<int32_t>(), ctx->ccsize.as<int32_t>(), ctx->ckey[cur].as<uint32_t>(),
            ctx->ccnt[cur].as<uint32_t>(), Q, ctx->ccctr.as<long long>(), (long long)kCompBudget);
        const cudaError_t le = cudaGetLastError();
        GS_CK(cudaEventSynchronize(ctx->ev_plan));
        const int ncomp = (int)plan[0], maxsz = (int)plan[1];
        const size_t csm = (size_t)plan[2];
        if (le == cudaSuccess) {
          GS_LAUNCHED("k_sweep_comp");
          if (ncomp == 0) return GS_OK;  // every cell isolated or frozen: Q rows are final (P3)
          if (csm <= kCompBudget && maxsz < 65535) return GS_OK;
          // (the launch was a no-op: some component does not fit a CTA)
        } else {
          ctx->comp_ok = false;  // cannot be launched here: the cluster sweeps from now on
          if (ncomp == 0) return GS_OK;
        }
      }
    }
  }
  constexpr size_t kBudget = 220 * 1024;
  const size_t smem = 4 * ((size_t)(m + 3) / 4 + 1) + 2 * (size_t)m;
  const int in_smem = (m < 65536 && smem <= kBudget) ? 1 : 0;
  static std::atomic<uint64_t> done_g{0}, done_f{0}, done_c{0};
  GS_CK(attr_once(done_g, ctx->device, gs::k_sweep_global<D>, (int)kBudget));
  const uint32_t dbg = ctx->sweep_flags;
  // the dataflow cluster sweep (no levels: a cell is updated as soon as its predecessors are).
  // measured: d = 5 (cfg3) 2.17 -> 1.85 ms per run; d = 3 (cfg5) 2.33 -> 2.45 ms (the per-hop
  // fence + remote release costs more than the level barrier saves when a cell has <= 27
  // terms), so d <= 3 keeps the level-synchronous sweep (test hooks force either)
  {
    int flow_sel = (dbg & GS_DEBUG_SWEEP_FLOW) ? 2 : (dbg & (GS_DEBUG_SWEEP_LEVELS | GS_DEBUG_SWEEP_SINGLE)) ? 0 : 1;
    if (const char* v = knob("GS_SWEEP_FLOW")) flow_sel = atoi(v);
    const int flow_sleep = knob("GS_FLOW_SLEEP") ? atoi(knob("GS_FLOW_SLEEP")) : 0;
    const int flow_fence = knob("GS_FLOW_FENCE") ? atoi(knob("GS_FLOW_FENCE")) : 0;
    if (ctx->flow_ok && (flow_sel > 1 || (flow_sel == 1 && D > 3))) {
      bool c16 = true;
      GS_CK(attr_once(done_f, ctx->device, gs::k_sweep_flow<D>, (int)kBudget, true, &c16));
      if (!c16) ctx->cluster16_ok = false;
      const int NC = ctx->cluster16_ok ? 16 : 8;
      const size_t fsm = gs::sweep_flow_smem<D>((int)((m + NC - 1) / NC));
      if (fsm <= kBudget) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)NC);
        lc.blockDim = dim3(512);
        lc.dynamicSmemBytes = fsm;
        lc.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)NC;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        const cudaError_t le = cudaLaunchKernelEx(
            &lc, gs::k_sweep_flow<D>, (int)m, KP, (const uint32_t*)lists,
            (const int32_t*)ctx->nbn.as<int32_t>(), (const int32_t*)ctx->nbe.as<int32_t>(),
            (const uint32_t*)ctx->ccnt[cur].as<uint32_t>(),
            (const uint32_t*)ctx->den.as<uint32_t>(), (const double*)ctx->rden.as<double>(), Q,
            ctx->errflag.as<int>(), flow_sleep, flow_fence, pinit);
        if (le == cudaSuccess) {
          GS_LAUNCHED("k_sweep_flow");
          return GS_OK;
        }
        cudaGetLastError();
        ctx->flow_ok = false;  // cannot be scheduled here: level-synchronous sweeps from now on
      }
    }
  }
  // the cluster sweep (NC CTAs on NC SMs, DSMEM pending counts and queues) when the owned
  // share of 3 words per cell fits each CTA; else the single-CTA sweep
  {
    int NC = (dbg & GS_DEBUG_SWEEP_SINGLE) || !ctx->cluster_ok ? 0 : 16;
    if (const char* v = knob("GS_SWEEP_CLUSTER")) NC = atoi(v);
    if (NC > 8) {
      bool c16 = true;
      GS_CK(attr_once(done_c, ctx->device, gs::k_sweep_cluster<D>, (int)kBudget, true, &c16));
      if (!c16) ctx->cluster16_ok = false;
      if (!ctx->cluster16_ok) NC = 8;
    } else if (NC >= 2) {
      GS_CK(attr_once(done_c, ctx->device, gs::k_sweep_cluster<D>, (int)kBudget, true));
    }
    const size_t csmem = gs::sweep_cluster_smem<D>((int)((m + NC - 1) / std::max(NC, 1)));
    if (NC >= 2 && csmem <= kBudget) {
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3((unsigned)NC);
      lc.blockDim = dim3(gs::sweep_cluster_threads<D>());
      lc.dynamicSmemBytes = gs::sweep_cluster_smem<D>((int)((m + NC - 1) / NC));
      lc.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = (unsigned)NC;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      long long* cprof = nullptr;
      const bool ctrace = knob("GS_TRACE_GLOBAL") != nullptr;
      if (ctrace) {
        GS_TRY(grow(ctx, ctx->dbg, 8 * (1000 * 16 * 5 + 8)));
        GS_CK(cudaMemsetAsync(ctx->dbg.p, 0, 8 * (1000 * 16 * 5 + 8), st));
        cprof = (long long*)ctx->dbg.p;
      }
      cudaError_t le = cudaLaunchKernelEx(&lc, gs::k_sweep_cluster<D>, (int)m, KP,
                                          (const uint32_t*)lists, (const int32_t*)ctx->nbn.as<int32_t>(),
                                          (const int32_t*)ctx->nbe.as<int32_t>(),
                                          (const uint32_t*)ctx->ccnt[cur].as<uint32_t>(),
                                          (const uint32_t*)ctx->den.as<uint32_t>(),
                                          (const double*)ctx->rden.as<double>(), Q, cprof, pinit);
      if (le == cudaSuccess) {
        GS_LAUNCHED("k_sweep_cluster");
        if (ctrace) {  // diagnostics: per-level split, max over CTAs
          std::vector<long long> h(1000 * 16 * 5 + 8);
          GS_CK(cudaMemcpyAsync(h.data(), cprof, 8 * h.size(), cudaMemcpyDeviceToHost, st));
          GS_CK(cudaStreamSynchronize(st));
          const int nl = (int)std::min<long long>(h[1000 * 16 * 5], 1000);
          double su = 0, sr = 0, sb = 0;
          for (int l = 0; l < nl; ++l) {
            long long wmax = 0, u = 0, r = 0, bq = 0, wsum = 0;
            for (int c = 0; c < NC; ++c) {
              const long long* p = &h[((size_t)l * 16 + c) * 5];
              wmax = std::max(wmax, p[0]);
              wsum += p[0];
              u = std::max(u, p[2] - p[1]);
              r = std::max(r, p[3] - p[2]);
              bq = std::max(bq, p[4] - p[3]);
            }
            su += u;
            sr += r;
            sb += bq;
            if (l < 6 || l % 25 == 0)
              fprintf(stderr, "csweep m %lld level %4d width %5lld (max/CTA %4lld) update %6lld release %6lld barrier %5lld\n",
                      (long long)m, l, wsum, wmax, u, r, bq);
          }
          fprintf(stderr, "csweep m %lld NC %d levels %d | mean max-over-CTA cycles: update %.0f release %.0f barrier %.0f\n",
                  (long long)m, NC, nl, su / std::max(nl, 1), sr / std::max(nl, 1), sb / std::max(nl, 1));
        }
        return GS_OK;
      }
      cudaGetLastError();  // a cluster this size cannot be scheduled: single-CTA sweep below
      if (NC > 8) ctx->cluster16_ok = false;
      else ctx->cluster_ok = false;
    }
  }
  long long* prof = nullptr;
  const bool trace = knob("GS_TRACE_GLOBAL") != nullptr;
  if (trace) {
    GS_TRY(grow(ctx, ctx->dbg, 8 * (2000 * 66 + 8)));
    GS_CK(cudaMemsetAsync(ctx->dbg.p, 0, 8 * (2000 * 66 + 8), st));
    prof = (long long*)ctx->dbg.p;
  }
  gs::k_sweep_global<D><<<1, gs::sweep_global_threads<D>(), in_smem ? smem : 0, st>>>(
      (int)m, KP, lists, ctx->nbn.as<int32_t>(), ctx->nbe.as<int32_t>(),
      ctx->ccnt[cur].as<uint32_t>(), ctx->den.as<uint32_t>(), ctx->rden.as<double>(), Q,
      ctx->lvl.as<unsigned>(), ctx->order.as<unsigned>(), in_smem, prof, pinit);
  GS_LAUNCHED("k_sweep_global");
  if (trace) {  // diagnostics: per-level update / release / barrier split of this sweep
    std::vector<long long> h(2000 * 66 + 8);
    GS_CK(cudaMemcpyAsync(h.data(), prof, 8 * h.size(), cudaMemcpyDeviceToHost, st));
    GS_CK(cudaStreamSynchronize(st));
    const int nl = (int)std::min<long long>(h[2000 * 66], 2000);
    const int nw = gs::sweep_global_threads<D>() / 32;
    double su = 0, sr = 0, sb = 0, sw = 0;
    for (int l = 0; l < nl; ++l) {
      const long long* p = &h[(size_t)l * 66];
      long long ue = 0, re = 0;
      for (int w = 0; w < nw; ++w) {
        ue = std::max(ue, p[2 + w]);
        re = std::max(re, p[34 + w]);
      }
      const long long nxt = l + 1 < nl ? h[(size_t)(l + 1) * 66 + 1] : re;
      su += ue - p[1];
      sr += re - ue;
      sb += nxt - re;
      sw += p[0];
      if (l < 8 || l % 20 == 0)
        fprintf(stderr, "gsweep m %lld level %4d width %5lld update %6lld release %6lld barrier %5lld\n",
                (long long)m, l, p[0], ue - p[1], re - ue, nxt - re);
    }
    fprintf(stderr, "gsweep m %lld levels %d mean width %.1f | mean cycles: update %.0f release %.0f barrier %.0f\n",
            (long long)m, nl, sw / std::max(nl, 1), su / std::max(nl, 1), sr / std::max(nl, 1),
            sb / std::max(nl, 1));
  }
  return GS_OK;
}

gs_status launch_global_sweep(gs_ctx* ctx, int d, int64_t m, int K,
                              const SweepHalo* halo = nullptr) {
  switch (d) {
#define GS_CASE(D) \
  case D:          \
    return launch_global_sweep_d<D>(ctx, m, K, halo);
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
#undef GS_CASE
  }
  return fail(ctx, GS_E_INVALID_PARAMETER, "d out of range");
}

// One iterate_once over all frames (frozen frames excluded).  Cells in buffer `cur`; the new
// cells land in buffer 1-cur.  Per-frame changed/adjacency/m/disp land in the f* arrays.
// defer_mnew: the new cell count stays on the device (the later kernels read it there, their
// grids sized for m) and the per-iteration accumulators are cleared by k_iter_pack, not here;
// *mnew_out = -1 and the caller reads the count with the rest of the iteration's state.
gs_status iterate(gs_ctx* ctx, int64_t m, int64_t* mnew_out, bool defer_mnew = false) {
  const GsBox& b = ctx->box;
  const int d = b.d;
  const int K = (int)ipow3(d);
  const int cur = ctx->cur, nxt = 1 - cur;
  const int64_t nf = b.nframes;
  cudaStream_t st = ctx->stream;
  if (!defer_mnew) {
    GS_CK(cudaMemsetAsync(ctx->fchanged.p, 0, sizeof(int32_t) * nf, st));
    GS_CK(cudaMemsetAsync(ctx->fadj.p, 0, sizeof(int32_t) * nf, st));
    GS_CK(cudaMemsetAsync(ctx->fm.p, 0, sizeof(int32_t) * nf, st));
    GS_CK(cudaMemsetAsync(ctx->fdisp.p, 0, sizeof(unsigned long long) * nf, st));
  }
  const unsigned mb = blocks_for(m, 256);
  if (d <= 6) {
    // (1) fixed-stride neighbour lists (all SMs), (2) the single-CTA Kahn sweep over L2
    GS_TRY(launch_global_sweep(ctx, d, m, K));
  } else {
  // (1) neighbour census -> scanned record offsets -> records (all SMs)
  gs::k_nbr_count<<<mb, 256, 0, st>>>((int)m, b, K, ctx->ckey[cur].as<uint32_t>(),
                                      ctx->idx.as<int32_t>(), ctx->fdone.as<int32_t>(),
                                      ctx->nbn.as<int32_t>(), ctx->nbe.as<int32_t>(),
                                      ctx->head.as<int32_t>(), ctx->sid.as<int32_t>(),
                                      ctx->fm.as<int32_t>());
  GS_LAUNCHED("k_nbr_count");
  int32_t* eoff = ctx->segstart.as<int32_t>();
  int32_t* loff = ctx->parent.as<int32_t>();  // parent is rewritten by k_seg later
  size_t tb = ctx->cub_tmp.bytes;
  GS_CK(cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, tb, ctx->head.as<int32_t>(), eoff, (int)m, st));
  GS_TRY(check_lib(ctx, "cub_scan_e"));
  tb = ctx->cub_tmp.bytes;
  GS_CK(cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, tb, ctx->sid.as<int32_t>(), loff, (int)m, st));
  GS_TRY(check_lib(ctx, "cub_scan_l"));
  int32_t tails[4];
  GS_CK(cudaMemcpyAsync(&tails[0], eoff + (m - 1), 4, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(&tails[1], ctx->head.as<int32_t>() + (m - 1), 4, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(&tails[2], loff + (m - 1), 4, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(&tails[3], ctx->sid.as<int32_t>() + (m - 1), 4, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaStreamSynchronize(st));
  const int64_t n_early = (int64_t)tails[0] + tails[1], n_late = (int64_t)tails[2] + tails[3];
  GS_TRY(grow(ctx, ctx->erec, 8 * std::max<int64_t>(1, n_early)));
  GS_TRY(grow(ctx, ctx->lprod, 8 * d * std::max<int64_t>(1, n_late)));
  GS_TRY(grow(ctx, ctx->rden, 8 * m));
  GS_TRY(grow(ctx, ctx->lvl, 4 * (m + 1)));
  GS_TRY(grow(ctx, ctx->lsucc, 4 * std::max<int64_t>(1, n_late)));
  GS_TRY(grow(ctx, ctx->order, 4 * m));
  gs::k_nbr_fill<<<mb, 256, 0, st>>>((int)m, b, K, ctx->ckey[cur].as<uint32_t>(),
                                     ctx->ccnt[cur].as<uint32_t>(), ctx->S[cur].as<double>(),
                                     ctx->idx.as<int32_t>(), ctx->nbn.as<int32_t>(), eoff, loff,
                                     ctx->erec.as<unsigned long long>(), ctx->lprod.as<double>(),
                                     ctx->lsucc.as<int32_t>(), ctx->den.as<uint32_t>(),
                                     ctx->rden.as<double>());
  GS_LAUNCHED("k_nbr_fill");
  // (2) the sweep: one CTA, DAG levels, level-synchronous exact Eq. (5)
  GS_TRY(launch_sweep_levels(ctx, d, m, eoff, loff));
  }
  gs::k_rehome<<<mb, 256, 0, ctx->stream>>>(
      (int)m, b, ctx->ckey[cur].as<uint32_t>(), ctx->S[cur].as<double>(), ctx->S1.as<double>(),
      ctx->fdone.as<int32_t>(), ctx->nkey.as<uint32_t>(), ctx->vals.as<uint32_t>(),
      ctx->fchanged.as<int32_t>(), ctx->fdisp.as<unsigned long long>(), ctx->errflag.as<int>());
  GS_LAUNCHED("k_rehome");
  const int kb = bits_for(b.vol_total);
  size_t tb = ctx->cub_tmp.bytes;
  GS_CK(cub::DeviceRadixSort::SortPairs(ctx->cub_tmp.p, tb, ctx->nkey.as<uint32_t>(),
                                        ctx->skey.as<uint32_t>(), ctx->vals.as<uint32_t>(),
                                        ctx->sval.as<uint32_t>(), (int)m, 0, kb, ctx->stream));
  GS_TRY(check_lib(ctx, "cub_sort_pairs"));
  gs::k_heads<<<mb, 256, 0, ctx->stream>>>((int)m, ctx->skey.as<uint32_t>(),
                                           ctx->head.as<int32_t>());
  GS_LAUNCHED("k_heads");
  tb = ctx->cub_tmp.bytes;
  GS_CK(cub::DeviceScan::InclusiveSum(ctx->cub_tmp.p, tb, ctx->head.as<int32_t>(),
                                      ctx->sid.as<int32_t>(), (int)m, ctx->stream));
  GS_TRY(check_lib(ctx, "cub_scan"));
  gs::k_seg<<<mb, 256, 0, ctx->stream>>>((int)m, ctx->head.as<int32_t>(), ctx->sid.as<int32_t>(),
                                         ctx->sval.as<uint32_t>(), ctx->parent.as<int32_t>(),
                                         ctx->segstart.as<int32_t>());
  GS_LAUNCHED("k_seg");
  int32_t mnew = (int32_t)m;  // (deferred: the grids' upper bound)
  const int32_t* mdev = defer_mnew ? ctx->sid.as<int32_t>() + (m - 1) : nullptr;
  if (!defer_mnew) {
    GS_CK(cudaMemcpyAsync(&mnew, ctx->sid.as<int32_t>() + (m - 1), sizeof(int32_t),
                          cudaMemcpyDeviceToHost, ctx->stream));
    GS_CK(cudaStreamSynchronize(ctx->stream));
  }
  const unsigned nb = blocks_for(mnew, 256);
  switch (d) {
#define GS_CASE(D)                                                                            \
  case D:                                                                                     \
    gs::k_fold<D><<<nb, 256, 0, ctx->stream>>>(                                               \
        mnew, (int)m, ctx->segstart.as<int32_t>(), ctx->skey.as<uint32_t>(),                 \
        ctx->sval.as<uint32_t>(), ctx->ccnt[cur].as<uint32_t>(), ctx->S1.as<double>(),       \
        ctx->ckey[nxt].as<uint32_t>(), ctx->ccnt[nxt].as<uint32_t>(), ctx->S[nxt].as<double>(), \
        mdev);                                                                                 \
    break;
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
    GS_CASE(7) GS_CASE(8) GS_CASE(9) GS_CASE(10) GS_CASE(11) GS_CASE(12)
#undef GS_CASE
  }
  GS_LAUNCHED("k_fold");
  gs::k_idx_clear<<<mb, 256, 0, ctx->stream>>>((int)m, ctx->ckey[cur].as<uint32_t>(),
                                               ctx->idx.as<int32_t>());
  GS_LAUNCHED("k_idx_clear");
  gs::k_idx_set<<<nb, 256, 0, ctx->stream>>>(mnew, ctx->ckey[nxt].as<uint32_t>(),
                                             ctx->idx.as<int32_t>(), mdev);
  GS_LAUNCHED("k_idx_set");
  switch (d) {
#define GS_ADJ(D)                                                                             \
  case D:                                                                                     \
    gs::k_adjacent<D><<<nb, 256, 0, ctx->stream>>>(mnew, b, K, ctx->ckey[nxt].as<uint32_t>(), \
                                                   ctx->idx.as<int32_t>(),                    \
                                                   ctx->fdone.as<int32_t>(),                  \
                                                   ctx->fadj.as<int32_t>(), mdev);            \
    break;
    GS_ADJ(1) GS_ADJ(2) GS_ADJ(3) GS_ADJ(4) GS_ADJ(5) GS_ADJ(6) GS_ADJ(7) GS_ADJ(8) GS_ADJ(9)
    GS_ADJ(10) GS_ADJ(11) GS_ADJ(12)
#undef GS_ADJ
  }
  GS_LAUNCHED("k_adjacent");
  ctx->cur = nxt;
  *mnew_out = defer_mnew ? -1 : mnew;
  return GS_OK;
}

// ---- K8 launch helpers
constexpr size_t kResidentSmemBudget = 224 * 1024;  // of 227 KB per CTA (static smem < 1 KB)
constexpr size_t kResidentStateMax = 160 * 1024;    // cell state may take at most this much

// Largest power-of-two cell capacity whose per-cell state fits kResidentStateMax; the rest of
// the budget holds the neighbour records (gs_resident.cuh falls back to slower sweep modes
// when a frame's records do not fit).
int resident_offs_bytes_host(int d) {
  switch (d) {
#define GS_CASE(D) \
  case D:          \
    return gs::resident_offs_bytes(D);
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
#undef GS_CASE
  }
  return 0;
}

int resident_capacity(int d) {
  int ms = 4096;
  while (ms > 32 && (size_t)ms * gs::resident_bytes_per_cell(d) > kResidentStateMax) ms >>= 1;
  return ms;
}

template <int D>
gs_status launch_resident_d(gs_ctx* ctx, unsigned grid, int threads, size_t smem,
                            const gs::ResidentArgs& ra) {
  static std::atomic<uint64_t> done{0};
  GS_CK(attr_once(done, ctx->device, gs::k_resident<D>, (int)kResidentSmemBudget + 1024));
  gs::k_resident<D><<<grid, threads, smem, ctx->stream>>>(ra);
  GS_LAUNCHED("k_resident");
  return GS_OK;
}

gs_status launch_resident(gs_ctx* ctx, int d, unsigned grid, int threads, size_t smem,
                          const gs::ResidentArgs& ra) {
  switch (d) {
#define GS_CASE(D) \
  case D:          \
    return launch_resident_d<D>(ctx, grid, threads, smem, ra);
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
    GS_CASE(7) GS_CASE(8) GS_CASE(9) GS_CASE(10) GS_CASE(11) GS_CASE(12)
#undef GS_CASE
  }
  return fail(ctx, GS_E_INVALID_PARAMETER, "d out of range");
}

// Readback area in pinned host memory: the control block's mirror (one D2H copy per run), then
// the per-iteration history (copied only when recorded).
struct Readback {
  int* err;          // 8 ints
  unsigned* ctr;     // 16
  int64_t* modes;    // 12
  int64_t* fswept;   // nf
  int32_t* fdone;    // nf
  int32_t* fiters;
  int32_t* fconv;
  int32_t* fk;
  int32_t* fout;
  int64_t* hm;       // nf * max_iter
  double* hd;        // nf * max_iter
};

gs_status map_readback(gs_ctx* ctx, int64_t nf_run, int max_iter, Readback* rb) {
  const int64_t nf = ctx->ctl_nf;  // the control block's layout (>= this run's frames)
  const size_t need = ctl_bytes(nf) + 16 * (size_t)nf_run * max_iter + 64;
  if (need > ctx->pin_bytes) {
    if (ctx->pin) cudaFreeHost(ctx->pin);
    ctx->pin = ctx->pin_dev = nullptr;
    ctx->pin_bytes = 0;
    GS_CK(cudaHostAlloc(&ctx->pin, need, cudaHostAllocMapped));
    GS_CK(cudaHostGetDevicePointer(&ctx->pin_dev, ctx->pin, 0));
    ctx->pin_bytes = need;
    ++ctx->alloc_gen;
  }
  char* p = (char*)ctx->pin;
  rb->err = (int*)p;
  rb->ctr = (unsigned*)(p + 32);
  rb->modes = (int64_t*)(p + 96);
  p += kCtlHeader;
  rb->fswept = (int64_t*)p;  p += 8 * (size_t)nf;
  rb->fdone = (int32_t*)p;   p += 4 * (size_t)nf;
  rb->fiters = (int32_t*)p;  p += 4 * (size_t)nf;
  rb->fconv = (int32_t*)p;   p += 4 * (size_t)nf;
  rb->fk = (int32_t*)p;      p += 4 * (size_t)nf;
  rb->fout = (int32_t*)p;    p += 4 * (size_t)nf;
  p = (char*)ctx->pin + ((ctl_bytes(nf) + 15) & ~size_t(15));
  rb->hm = (int64_t*)p;      p += 8 * (size_t)nf_run * max_iter;
  rb->hd = (double*)p;
  return GS_OK;
}

// K7 grid: frames along y, ~8 CTAs of 256 per SM in total
dim3 label_grid(gs_ctx* ctx, int64_t n, int64_t nf) {
  const int64_t y = std::min<int64_t>(nf, 65535);
  const int64_t total = (int64_t)ctx->num_sms * 8;
  const int64_t x = std::max<int64_t>(1, std::min<int64_t>((n + 2047) / 2048, (total + y - 1) / y));
  return dim3((unsigned)x, (unsigned)y);
}

// K8 over every frame, then labels; results copied to the pinned readback area; one sync.
// deferrable: the launch is optimistic (smem sized from the shape cache) and K8 may refuse.
bool graph_safe(const void* p);

gs_status launch_tail(gs_ctx* ctx, const gs_config* cfg, int64_t nf, int64_t ntot, int d,
                      int ms_run, bool deferrable, bool initial_ranges, int32_t* user_labels,
                      bool dev_out, bool rec, const Readback& rb) {
  cudaStream_t st = ctx->stream;
  const int ms_cap = resident_capacity(d);
  ms_run = std::min(std::max(ms_run, 32), ms_cap);
  // the sweep itself uses 128 threads (named barrier); the parallel phases loop over cells, so
  // 256 threads keep block barriers cheap up to ~1K cells
  // the sweep runs one warp per cell, so a level of up to T/32 cells completes in one round;
  // fewer threads when frames share an SM
  const int threads = nf > ctx->num_sms ? 256 : 512;
  const int64_t per_sm = std::min<int64_t>(4, std::max<int64_t>(1, (nf + ctx->num_sms - 1) / ctx->num_sms));
  const size_t budget = kResidentSmemBudget / per_sm - (per_sm > 1 ? 1024 : 0);
  const size_t state = (size_t)ms_run * gs::resident_bytes_per_cell(d);
  // the box's frame volume is host-known only on the synchronous path; the optimistic path
  // uses the cached choice
  const int64_t vf = deferrable ? ctx->shape_vol_frame : ctx->box.vol_frame;
  const size_t sidx = (vf * 2 <= 48 * 1024) ? ((size_t)vf * 2 + 15) & ~size_t(15) : 0;
  const size_t offs_bytes = (size_t)resident_offs_bytes_host(d) + gs::resident_fixed_bytes(d);
  const size_t fixed = state + sidx + offs_bytes;
  const size_t pool_bytes = budget > fixed + 1024 ? budget - fixed : 1024;
  unsigned* cnt32 = ctx->counters.as<unsigned>();
  // K8 owns the global index from here on (it clears or re-keys each frame's entries and
  // leaves the grid clean)
  const int fin = 1 - ctx->cur;
  gs::ResidentArgs ra;
  ra.ms = ms_run;
  ra.pool_bytes = (int)(pool_bytes & ~size_t(15));
  ra.max_iter = cfg->max_iter;
  ra.record = rec ? 1 : 0;
  ra.ckey = ctx->ckey[ctx->cur].as<uint32_t>();
  ra.ccnt = ctx->ccnt[ctx->cur].as<uint32_t>();
  ra.S = ctx->S[ctx->cur].as<double>();
  // current ranges: the initial ones (ffirst[f + 1] - ffirst[f]) unless the global path ran
  ra.ffirst = initial_ranges ? ctx->ifirst.as<int32_t>() : ctx->ffirst.as<int32_t>();
  ra.fcount = initial_ranges ? nullptr : ctx->fcount.as<int32_t>();
  ra.ifirst = ctx->ifirst.as<int32_t>();
  ra.initkey = ctx->initkey.as<uint32_t>();
  ra.lab = ctx->lab.as<int32_t>();
  ra.fdone = ctx->fdone.as<int32_t>();
  ra.fiters = ctx->fiters.as<int32_t>();
  ra.fconv = ctx->fconv.as<int32_t>();
  ra.fk = ctx->fk.as<int32_t>();
  ra.fout = ctx->fout.as<int32_t>();
  ra.fswept = ctx->fswept.as<int64_t>();
  ra.okey = ctx->ckey[fin].as<uint32_t>();
  ra.ocnt = ctx->ccnt[fin].as<uint32_t>();
  ra.oS = ctx->S[fin].as<double>();
  ra.root = ctx->root.as<int32_t>();
  ra.hist_m = ctx->hist.as<int64_t>();
  ra.hist_d = (double*)(ctx->hist.as<int64_t>() + nf * cfg->max_iter);
  ra.err = ctx->errflag.as<int>();
  ra.mode_count = ctx->modes.as<int64_t>();
  // per-phase cycle counters cost a global atomic per phase: opt-in diagnostics only
  ra.prof = knob("GS_PROF") ? (long long*)(ctx->modes.as<int64_t>() + 4) : nullptr;
  ra.gidx = ctx->idx.as<int32_t>();
  ra.sidx_bytes = (int)sidx;
  ra.trace = nullptr;
  if (knob("GS_TRACE_LEVELS")) {
    GS_TRY(grow(ctx, ctx->dbg, 8 * 12000));
    GS_CK(cudaMemsetAsync(ctx->dbg.p, 0, 8 * 12000, st));
    ra.trace = (long long*)ctx->dbg.p;
  }
  ra.deferrable = deferrable ? 1 : 0;
  ra.deferred = (int*)(cnt32 + 4);
  ra.pbox = ctx->dbox.as<GsBox>();
  GS_TRY(launch_resident(ctx, d, (unsigned)nf, threads, fixed + ra.pool_bytes, ra));
  GS_TRY(rec_event(ctx, 3));
  // ---- labels: K8 wrote lab[initial cell key] = final frame-local id; label[p] = lab[slot[p]]
  //      (straight into pinned caller memory when it is graph-safe host memory)
  int32_t* dlabels = user_labels;
  // (large label arrays leave by DMA: the copy engine's bursts beat SM-issued stores over the
  // bus, as for the inputs past kZeroCopyMaxBytes)
  const bool direct = dev_out || (graph_safe(user_labels) &&
                                  sizeof(int32_t) * (size_t)ntot <= (size_t(16) << 20));
  if (!direct) {
    GS_TRY(grow(ctx, ctx->labels, sizeof(int32_t) * ntot));
    dlabels = ctx->labels.as<int32_t>();
  }
  auto* klab = vf > 65536 ? gs::k_label<true> : gs::k_label<false>;  // (tuning only, see K7)
  klab<<<label_grid(ctx, ntot / nf, nf), 256, 0, st>>>(
      ntot / nf, nf, ctx->slot.p, ctx->dbox.as<GsBox>(), ctx->lab.as<int32_t>(), dlabels,
      ctx->ctl.as<unsigned>(), (unsigned*)ctx->pin_dev, (int)(ctl_bytes(ctx->ctl_nf) / 4),
      (int)(ctl_zero_bytes(ctx->ctl_nf) / 4));
  GS_LAUNCHED("k_label");
  ctx->ctl_clean = true;  // K7 re-zeroes the control block (stream order: before any later use)
  GS_TRY(rec_event(ctx, 4));
  if (!direct)
    GS_CK(cudaMemcpyAsync(user_labels, dlabels, sizeof(int32_t) * ntot, cudaMemcpyDeviceToHost,
                          st));
  GS_TRY(rec_event(ctx, 5));
  if (rec) {
    GS_CK(cudaMemcpyAsync(rb.hm, ra.hist_m, 8 * nf * cfg->max_iter, cudaMemcpyDeviceToHost, st));
    GS_CK(cudaMemcpyAsync(rb.hd, ra.hist_d, 8 * nf * cfg->max_iter, cudaMemcpyDeviceToHost, st));
  }
  return GS_OK;  // the caller synchronises (or captures this sequence into a graph)
}

// GS_TRACE_LEVELS diagnostics: per-level timeline of frame 0's first sweep and per-iteration
// phase timeline of frame 0 (K8 writes them into ctx->dbg)
void dump_trace(gs_ctx* ctx) {
  if (!knob("GS_TRACE_LEVELS") || !ctx->dbg.p) return;
  {
      std::vector<long long> tr(8 * 512);
      cudaMemcpy(tr.data(), ctx->dbg.p, 8 * 8 * 512, cudaMemcpyDeviceToHost);
      std::vector<long long> tp9(256);
      cudaMemcpy(tp9.data(), (long long*)ctx->dbg.p + 9000, 8 * 256, cudaMemcpyDeviceToHost);
      std::vector<long long> ti(512);
      cudaMemcpy(ti.data(), (long long*)ctx->dbg.p + 4096, 8 * 512, cudaMemcpyDeviceToHost);
      std::vector<long long> ts(1024);
      cudaMemcpy(ts.data(), (long long*)ctx->dbg.p + 9700, 8 * 1024, cudaMemcpyDeviceToHost);
      for (int t = 0; t < 64; ++t) {
        if (!ti[8 * t + 7]) continue;  // (iterations run on the global path have no stamps)
        const long long* y = &ts[16 * t];
        const long long* x = &ti[8 * t];
        fprintf(stderr, "sub %2d lists: top->loop %5lld loop(t0) %5lld barrier %5lld | fold: heads->scan %5lld seg %5lld fold(t0) %5lld roots+retire %5lld barrier %5lld\n",
                t, y[0] - x[7], y[1] - y[0], x[0] - y[1], y[3] - y[2], y[4] - y[3], y[5] - y[4], y[6] - y[5], y[7] - y[6]);
      }
      for (int t = 0; t < 64; ++t) {
        if (!ti[8 * t + 7]) continue;
        const long long* x = &ti[8 * t];
        const long long* y = &((const long long*)tp9.data())[4 * t];
        fprintf(stderr, "iter %2d m %5lld lists %6lld sweep %6lld (levels %4lld: relax %6lld sort %5lld) rehome %6lld sort %6lld fold %6lld adj %6lld\n",
                t, x[6], x[0] - x[7], x[1] - x[0], y[2], y[0] ? y[0] - x[0] : 0, y[1] - y[0], x[2] - x[1], x[3] - x[2], x[4] - x[3], x[5] - x[4]);
      }
      std::vector<long long> tp(8 * 512);
      cudaMemcpy(tp.data(), (long long*)ctx->dbg.p + 6000, 8 * 8 * 512, cudaMemcpyDeviceToHost);
      for (int l = 0; l < 512 && (tr[8 * l + 1] || tr[8 * l]); ++l)
        fprintf(stderr, "level %3d upd %5lld width %3lld n %3lld e %3lld | meta %4lld vals %4lld chain %4lld div+st %4lld bar %4lld gap %4lld\n", l, tr[8 * l + 1],
                tr[8 * l + 3], tr[8 * l + 4], tr[8 * l + 5], tp[8 * l], tp[8 * l + 1], tp[8 * l + 2],
                tp[8 * l + 3], tp[8 * l + 5] - tp[8 * l + 4] - tp[8 * l] - tp[8 * l + 1] - tp[8 * l + 2] - tp[8 * l + 3],
                l ? tp[8 * l + 4] - tp[8 * (l - 1) + 5] : 0);
      }
}

// Host memory the graph may copy from/to without staging: pinned or device-visible.
bool graph_safe(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeDevice ||
         at.type == cudaMemoryTypeManaged;
}

// Pinned inputs up to this size are read by K1 over the bus instead of copied (cfg2: e2e
// 728 -> 755 M points/s); above it the copy engine wins (cfg4, 943 MB: 3.15 -> 2.96 G).
constexpr size_t kZeroCopyMaxBytes = size_t(16) << 20;

// The device address of pinned host memory a kernel may read directly, or null.
const void* pinned_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

__global__ void k_epoch_bump(unsigned* e) { *e += 1u; }

// The front of gs_shard_run: every rank's partial cells (host) -> the dense grid of the
// global box -> compaction, leaving the same device state launch_nscale leaves after binning
// the whole cloud (the shard's slot[] is still there from gs_shard_bin).
gs_status launch_shard_front(gs_ctx* ctx, int d) {
  cudaStream_t st = ctx->stream;
  const int64_t m = ctx->shard_m;
  GS_TRY(rec_event(ctx, 0));
  GS_TRY(rec_event(ctx, 1));
  GS_TRY(grow(ctx, ctx->pkeys, 4 * std::max<int64_t>(m, 1)));
  GS_TRY(grow(ctx, ctx->pcounts, 4 * std::max<int64_t>(m, 1)));
  GS_TRY(grow(ctx, ctx->psums, 8 * d * std::max<int64_t>(m, 1)));
  GS_TRY(ensure_cells(ctx, std::min<int64_t>(m, ctx->box.vol_total), d));
  GS_CK(cudaMemcpyAsync(ctx->pkeys.p, ctx->shard_keys, 4 * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->pcounts.p, ctx->shard_counts, 4 * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->psums.p, ctx->shard_sums, 8 * d * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemsetAsync(ctx->ctl.p, 0, ctl_zero_bytes(ctx->ctl_nf), st));
  GS_CK(cudaMemcpyAsync(ctx->dbox.p, &ctx->box, sizeof(GsBox), cudaMemcpyHostToDevice, st));
  GS_TRY(rec_event(ctx, 6));
  gs::k_scatter_partials<<<blocks_for(m, 256, (int64_t)ctx->num_sms * 8), 256, 0, st>>>(
      m, d, ctx->pkeys.as<uint32_t>(), ctx->pcounts.as<uint32_t>(),
      ctx->psums.as<long long>(), ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>());
  GS_LAUNCHED("k_scatter_partials");
  GS_TRY(rec_event(ctx, 7));
  k_epoch_bump<<<1, 1, 0, st>>>(ctx->epoch_dev.as<unsigned>());
  GS_LAUNCHED("k_epoch_bump");
  unsigned* cnt32 = ctx->counters.as<unsigned>();
  const unsigned tg = (unsigned)std::min<int64_t>(ctx->box.vol_total / gs::kOccTile + 1,
                                                  (int64_t)ctx->num_sms * 4);
  gs::k_occ<<<tg, 256, 0, st>>>(
      ctx->dbox.as<GsBox>(), ctx->epoch_dev.as<unsigned>(), ctx->tiles.as<unsigned long long>(),
      cnt32 + 5, cnt32, ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>(),
      ctx->ckey[0].as<uint32_t>(), ctx->ccnt[0].as<uint32_t>(), ctx->S[0].as<double>(),
      ctx->idx.as<int32_t>(), ctx->root.as<int32_t>(), ctx->initkey.as<uint32_t>(),
      ctx->ifirst.as<int32_t>(), ctx->errflag.as<int>());
  GS_LAUNCHED("k_occ");
  GS_TRY(rec_event(ctx, 2));
  return GS_OK;
}

// opt-in host-side timeline of one run (GS_HOST_PROF): prep / launch / wait / results, in us
struct HostProf {
  bool on = knob("GS_HOST_PROF") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), t = t0;
  double seg[4] = {0, 0, 0, 0};
  void lap(int i) {
    if (!on) return;
    auto n = std::chrono::steady_clock::now();
    seg[i] += std::chrono::duration<double, std::micro>(n - t).count();
    t = n;
  }
  ~HostProf() {
    if (on) fprintf(stderr, "host prof: prep %.1f launch %.1f wait %.1f results %.1f us\n", seg[0], seg[1], seg[2], seg[3]);
  }
};

int img_width(const gs_input* in) {
  return (in->dtype == GS_U8 && in->d == 5) ? in->reserved : 0;
}

gs_status run_impl(gs_ctx* ctx, const gs_input* in, const gs_config* cfg, gs_result* out) {
  HostProf hp;
  GS_TRY(validate(in, cfg));
  if (!ctx->shard_front) ctx->img_w = img_width(in);
  if (!out || !out->labels || !out->k || !out->iterations || !out->converged)
    return fail(ctx, GS_E_INVALID_PARAMETER, "null result buffer");
  const int d = in->d;
  const int64_t n = in->n, nf = in->batch, ntot = n * nf;
  const bool rec = (cfg->flags & GS_RECORD_HISTORY) != 0;
  const bool dev_out = (cfg->flags & GS_DEVICE_OUTPUTS) != 0;
  const bool force_global = (cfg->flags & GS_DEBUG_GLOBAL_PATH) != 0;
  ctx->have_run = false;
  ctx->grouped = false;
  ctx->stats = gs_stats{};
  ctx->stats_times_pending = false;
  ctx->ev_mask = ((cfg->flags & GS_TIME_PHASES) ? 0x3ffu : 0u) |
                 ((cfg->flags & GS_TIME_KERNEL) ? 0xc0u : 0u);
  ctx->cur = 0;
  cudaGetLastError();  // a stale error from an unrelated earlier call must not fail this run
  cudaStream_t st = ctx->stream;
  GS_TRY(grow(ctx, ctx->errflag, 32));
  GS_TRY(grow(ctx, ctx->counters, 64));
  GS_TRY(ensure_frames(ctx, nf));
  GS_TRY(grow(ctx, ctx->hist, (sizeof(int64_t) + sizeof(double)) * nf * cfg->max_iter));
  GS_TRY(grow(ctx, ctx->modes, sizeof(int64_t) * 12));
  Readback rb;
  GS_TRY(map_readback(ctx, nf, cfg->max_iter, &rb));
  ctx->hist_m.assign(rec ? nf : 0, {});
  ctx->hist_d.assign(rec ? nf : 0, {});
  if (!in->on_device) GS_TRY(grow(ctx, ctx->pts, input_bytes(in)));
  const void* dpts = in->on_device ? in->points : ctx->pts.p;
  int64_t vol_hint = 0;  // the cached shape's grid volume (sizes the compaction launch)
  ctx->sweep_flags = cfg->flags & (GS_DEBUG_SWEEP_FLOW | GS_DEBUG_SWEEP_LEVELS | GS_DEBUG_SWEEP_SINGLE);
  // the predicted key box (no bounds pass): the last box at this (d, dtype, h, image width),
  // re-based to this call's point and frame counts (not for the shard / debug entry points;
  // a pinned input small enough for the zero-copy pass still runs K1, as the copy)
  GsBox pbox_run{};
  const GsBox* pb = nullptr;
  auto choose_pbox = [&]() -> gs_status {
    pb = nullptr;
    if (ctx->shard_front || force_global || !ctx->pbox_valid || ctx->pbox_d != d ||
        ctx->pbox_dtype != in->dtype || ctx->pbox_h != cfg->h || ctx->pbox_w != ctx->img_w)
      return GS_OK;
    pbox_run = ctx->pbox;
    pbox_run.n = n;
    pbox_run.nframes = nf;
    pbox_run.F = gs_fixed_shift(n, cfg->h);
    pbox_run.scale = std::ldexp(1.0, pbox_run.F);
    pbox_run.inv_scale = std::ldexp(1.0, -pbox_run.F);
    pbox_run.vol_total = pbox_run.vol_frame * nf;
    if (pbox_run.vol_total > kMaxDenseCells) return GS_OK;
    GS_TRY(ensure_dense(ctx, pbox_run.vol_total, d));
    pb = &pbox_run;
    return GS_OK;
  };
  // K2 binned against the predicted box and flagged a point outside it (128) or a non-finite
  // coordinate (1): K3 skipped, so the grid holds K2's partial sums -- clear them
  auto clear_predicted = [&]() -> gs_status {
    GS_CK(cudaMemsetAsync(ctx->cnt.p, 0, sizeof(uint32_t) * pbox_run.vol_total, st));
    GS_CK(cudaMemsetAsync(ctx->qs.p, 0, sizeof(unsigned long long) * pbox_run.vol_total * d, st));
    GS_CK(cudaStreamSynchronize(st));
    ctx->pbox_valid = false;
    ctx->pbox_gen++;
    pb = nullptr;
    return GS_OK;
  };
  auto enqueue_front = [&]() -> gs_status {  // points to HBM, then the n-scale phase
    if (ctx->shard_front) return launch_shard_front(ctx, d);
    GS_TRY(rec_event(ctx, 0));
    // pinned caller points: K1 reads them over the bus and stores the device copy (the copy
    // and the bounds pass overlap; no copy node); pageable points: an explicit copy
    ctx->host_src = nullptr;
    if (!in->on_device) {
      // (large inputs go by DMA: measured, K1's bus reads lose to the copy engine past ~MBs)
      if (input_bytes(in) <= kZeroCopyMaxBytes) ctx->host_src = pinned_device_ptr(in->points);
      if (!ctx->host_src)
        GS_CK(cudaMemcpyAsync(ctx->pts.p, in->points, input_bytes(in), cudaMemcpyHostToDevice, st));
    }
    GS_TRY(rec_event(ctx, 1));
    const gs_status sf = launch_nscale(ctx, dpts, in->dtype, d, n, nf, cfg->h, vol_hint,
                                       pb);
    ctx->host_src = nullptr;
    GS_TRY(sf);
    GS_TRY(rec_event(ctx, 2));
    return GS_OK;
  };
  const gs_ctx::ShapeKey key{n, nf, d, in->dtype, cfg->h, cfg->max_iter, ctx->img_w};
  gs_ctx::ShapeEntry* sent = nullptr;  // this shape's cache entry, if any
  for (auto& e : ctx->shapes)
    if (e.ms > 0 && e.key == key) sent = &e;
  if (sent) {
    ctx->shape = key;
    ctx->shape_ms = sent->ms;
    ctx->shape_box = sent->box;
    ctx->shape_vol_frame = sent->vol_frame;
    sent->used = ++ctx->shape_tick;
  } else {
    ctx->shape_ms = 0;
  }
  std::vector<int32_t> g_iters(nf, 0);
  int64_t swept = 0;
  GS_TRY(choose_pbox());
  if (!force_global && !ctx->shard_front && ctx->shape_ms > 0 && key == ctx->shape && pb) {
    // ---- optimistic path: the whole run with no host round trip, replayed from a CUDA graph
    //      when the caller's buffers allow it (pinned or device memory)
    const bool graphed = ctx->use_graphs && (in->on_device || graph_safe(in->points)) &&
                         (dev_out || graph_safe(out->labels));
    vol_hint = ctx->shape_vol_frame * nf;
    auto enqueue_all = [&]() -> gs_status {
      GS_TRY(enqueue_front());
      return launch_tail(ctx, cfg, nf, ntot, d, ctx->shape_ms, true, true, out->labels, dev_out,
                         rec, rb);
    };
    if (graphed) {
      GS_TRY(clean_ctl(ctx));  // the graph has no memset node: it starts from a clean block
      const gs_ctx::GraphKey gk{key, in->points, out->labels, cfg->flags, in->on_device,
                                ctx->alloc_gen, pb ? ctx->pbox_gen : ~0ull};
      if (!(ctx->gexec && ctx->gkey == gk)) {
        if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
        const int64_t l0 = ctx->stats.kernel_launches;
        GS_CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
        const gs_status s = enqueue_all();
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(st, &graph);
        if (s != GS_OK) {
          if (graph) cudaGraphDestroy(graph);
          return s;
        }
        GS_CK(ce);
        const cudaError_t ie = cudaGraphInstantiate(&ctx->gexec, graph, 0);
        cudaGraphDestroy(graph);
        GS_CK(ie);
        ctx->gkey = gk;
        ctx->gkey.gen = ctx->alloc_gen;  // buffers (re)allocated while capturing belong to it
        ctx->graph_launches = ctx->stats.kernel_launches - l0;
      }
      hp.lap(0);
      GS_CK(cudaGraphLaunch(ctx->gexec, st));
      hp.lap(1);
      ctx->stats.kernel_launches = ctx->graph_launches;
    } else {
      GS_TRY(enqueue_all());
    }
    GS_CK(cudaStreamSynchronize(st));
    hp.lap(2);
    dump_trace(ctx);
    if (pb && (rb.err[0] & (1 | 128))) {
      GS_TRY(clear_predicted());
      if (rb.err[0] & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
    }
    if (rb.err[0] & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
    if (rb.err[0] & 64) return fail(ctx, GS_E_KEY_RANGE, "cell keys exceed the int64 key range");
    if (rb.err[0] & 4) return fail(ctx, GS_E_INTERNAL_INVARIANT, "centroid left the key box");
    if (rb.err[0] & 8) return fail(ctx, GS_E_INTERNAL_INVARIANT, "sweep schedule watchdog fired");
    if (rb.err[0] & 128) {
      // a point outside the predicted box: redo the run with the bounds pass (below)
    } else if ((rb.err[0] & 32) || rb.ctr[4] != 0) {  // grid too small / a frame too big: redo it
      ctx->shape_ms = 0;                        // synchronously below
      if (sent) sent->ms = 0;
      if (rb.err[0] & 32) GS_TRY(grow_dense_for(ctx, *(long long*)(rb.err + 2), d));
    } else {
      goto results;
    }
  }
  for (int attempt = 0;; ++attempt) {
    if (attempt > 3) return fail(ctx, GS_E_INTERNAL_INVARIANT, "could not size the cell grid");
    vol_hint = 0;
    GS_TRY(enqueue_front());
    // ---- synchronous path: the host sees the initial cells and drives the global path
    int hdr[8];
    unsigned ctr[16];
    GS_CK(cudaMemcpyAsync(hdr, ctx->errflag.p, 32, cudaMemcpyDeviceToHost, st));
    GS_CK(cudaMemcpyAsync(ctr, ctx->counters.p, 64, cudaMemcpyDeviceToHost, st));
    GS_CK(cudaMemcpyAsync(&ctx->box, ctx->dbox.p, sizeof(GsBox), cudaMemcpyDeviceToHost, st));
    GS_CK(cudaStreamSynchronize(st));
    if (pb && (hdr[0] & (1 | 128))) {
      GS_TRY(clear_predicted());
      if (hdr[0] & 128) continue;  // redo with the bounds pass
    }
    if (hdr[0] & 32) {
      GS_TRY(grow_dense_for(ctx, *(long long*)(hdr + 2), d));
      continue;
    }
    if (hdr[0] & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
    if (hdr[0] & 64) return fail(ctx, GS_E_KEY_RANGE, "cell keys exceed the int64 key range");
    if (hdr[0] & 2) return fail(ctx, GS_E_INTERNAL_INVARIANT, "a point's key left the key box");
    const int64_t m0 = ctr[0];
    const GsBox& b = ctx->box;
    // (a) global path (K4/K5 kernels, host-driven) while some live frame has more active
    //     cells than one CTA's shared memory holds; (b) then K8 runs every remaining
    //     iteration of every frame on the device.
    ctx->h_done.assign(nf, 0);
    ctx->h_iters.assign(nf, 0);
    ctx->h_conv.assign(nf, 0);
    ctx->hist_m.assign(rec ? nf : 0, {});
    ctx->hist_d.assign(rec ? nf : 0, {});
    std::vector<int32_t> fch(nf), fadj(nf), fm(nf), fcnt(nf);
    std::vector<unsigned long long> fdisp(nf);
    {
      std::vector<int32_t> f0(nf + 1);
      GS_CK(cudaMemcpyAsync(f0.data(), ctx->ifirst.p, sizeof(int32_t) * (nf + 1),
                            cudaMemcpyDeviceToHost, st));
      GS_CK(cudaStreamSynchronize(st));
      for (int64_t f = 0; f < nf; ++f) fcnt[f] = f0[f + 1] - f0[f];
    }
    int64_t m = m0, live = nf;
    int iter = 0;
    const int ms_cap = resident_capacity(d);
    auto max_live = [&]() {
      int64_t mx = 0;
      for (int64_t f = 0; f < nf; ++f)
        if (!ctx->h_done[f]) mx = std::max<int64_t>(mx, fcnt[f]);
      return mx;
    };
    // one packed device->host copy per iteration (new cell count, error bits, per-frame state):
    // the accumulators start clean here and k_iter_pack leaves them clean
    GS_CK(cudaMemsetAsync(ctx->fchanged.p, 0, sizeof(int32_t) * nf, st));
    GS_CK(cudaMemsetAsync(ctx->fadj.p, 0, sizeof(int32_t) * nf, st));
    GS_CK(cudaMemsetAsync(ctx->fm.p, 0, sizeof(int32_t) * nf, st));
    GS_CK(cudaMemsetAsync(ctx->fdisp.p, 0, sizeof(unsigned long long) * nf, st));
    const size_t pack_bytes = 16 + 24 * (size_t)nf;
    GS_TRY(ensure_hpin(ctx, 64 + pack_bytes));
    GS_TRY(grow(ctx, ctx->iterpack, pack_bytes));
    int32_t* hpack = (int32_t*)((char*)ctx->hpin + 64);
    while (live > 0 && (force_global || max_live() > ms_cap)) {
      int64_t mnew = 0;
      GS_TRY(iterate(ctx, m, &mnew, true));
      const int32_t* mdev = ctx->sid.as<int32_t>() + (m - 1);
      gs::k_compose<<<blocks_for(m0, 256), 256, 0, st>>>((int)m0, ctx->parent.as<int32_t>(),
                                                          ctx->root.as<int32_t>());
      GS_LAUNCHED("k_compose");
      gs::k_frame_ranges<<<blocks_for(m, 256), 256, 0, st>>>(
          (int)m, b.vol_frame, ctx->ckey[ctx->cur].as<uint32_t>(),
          ctx->ffirst.as<int32_t>(), ctx->fcount.as<int32_t>(), mdev);
      GS_LAUNCHED("k_frame_ranges");
      gs::k_iter_pack<<<blocks_for(nf, 256), 256, 0, st>>>(
          nf, ctx->ffirst.as<int32_t>(), ctx->fcount.as<int32_t>(), ctx->fchanged.as<int32_t>(),
          ctx->fadj.as<int32_t>(), ctx->fm.as<int32_t>(), ctx->fdisp.as<unsigned long long>(),
          mdev, ctx->errflag.as<int>(), ctx->iterpack.as<int32_t>());
      GS_LAUNCHED("k_iter_pack");
      GS_CK(cudaMemcpyAsync(hpack, ctx->iterpack.p, pack_bytes, cudaMemcpyDeviceToHost, st));
      GS_CK(cudaStreamSynchronize(st));
      mnew = hpack[0];
      const int err = hpack[1];
      std::memcpy(fch.data(), hpack + 4, 4 * (size_t)nf);
      std::memcpy(fadj.data(), hpack + 4 + nf, 4 * (size_t)nf);
      std::memcpy(fm.data(), hpack + 4 + 2 * nf, 4 * (size_t)nf);
      std::memcpy(fcnt.data(), hpack + 4 + 3 * nf, 4 * (size_t)nf);
      std::memcpy(fdisp.data(), hpack + 4 + 4 * nf, 8 * (size_t)nf);
      if (err & 8) return fail(ctx, GS_E_INTERNAL_INVARIANT, "sweep dataflow watchdog fired");
      if (err & 4) return fail(ctx, GS_E_INTERNAL_INVARIANT, "centroid left the key box");
      ++iter;
      bool newly_done = false;
      for (int64_t f = 0; f < nf; ++f) {
        if (ctx->h_done[f]) continue;
        swept += fm[f];
        if (rec) {
          double dsp;
          std::memcpy(&dsp, &fdisp[f], sizeof(double));
          ctx->hist_m[f].push_back(fm[f]);
          ctx->hist_d[f].push_back(dsp);
        }
        ctx->h_iters[f] = iter;
        const bool conv = !fadj[f] || !fch[f];
        if (conv || iter >= cfg->max_iter) {
          ctx->h_done[f] = 1;
          ctx->h_conv[f] = conv ? 1 : 0;
          --live;
          newly_done = true;
        }
      }
      m = mnew;
      if (newly_done)
        GS_CK(cudaMemcpyAsync(ctx->fdone.p, ctx->h_done.data(), sizeof(int32_t) * nf,
                              cudaMemcpyHostToDevice, st));
    }
    g_iters = ctx->h_iters;
    GS_CK(cudaMemcpyAsync(ctx->fiters.p, ctx->h_iters.data(), sizeof(int32_t) * nf,
                          cudaMemcpyHostToDevice, st));
    GS_CK(cudaMemcpyAsync(ctx->fconv.p, ctx->h_conv.data(), sizeof(int32_t) * nf,
                          cudaMemcpyHostToDevice, st));
    const int64_t ml = std::max<int64_t>(1, max_live());
    int ms_run = 32;
    while (ms_run < ml) ms_run <<= 1;
    ms_run = std::min(ms_run, ms_cap);
    if (iter == 0 && !force_global && !ctx->shard_front) {  // later runs go optimistic
      ctx->shape = key;
      ctx->shape_ms = std::min(ms_cap, 2 * ms_run);  // headroom for data-dependent m0
      ctx->shape_box = b;
      ctx->shape_vol_frame = b.vol_frame;
      gs_ctx::ShapeEntry* e = sent;
      if (!e) {  // least recently used entry
        e = &ctx->shapes[0];
        for (auto& x : ctx->shapes)
          if (x.used < e->used) e = &x;
      }
      *e = gs_ctx::ShapeEntry{key, ctx->shape_ms, b, b.vol_frame, ++ctx->shape_tick};
    }
    GS_TRY(launch_tail(ctx, cfg, nf, ntot, d, ms_run, false, iter == 0, out->labels, dev_out,
                       rec, rb));
    GS_CK(cudaStreamSynchronize(st));
    dump_trace(ctx);
    if (rb.err[0] & 8) return fail(ctx, GS_E_INTERNAL_INVARIANT, "sweep schedule watchdog fired");
    if (rb.err[0] & 16)
      return fail(ctx, GS_E_INTERNAL_INVARIANT, "frame exceeded the resident capacity");
    if (rb.err[0] & 4) return fail(ctx, GS_E_INTERNAL_INVARIANT, "centroid left the key box");
    break;
  }
results:
  ctx->cur = 1 - ctx->cur;  // K8 wrote the final cells to the other buffer
  if (!ctx->shard_front && !force_global) {  // this run's key box predicts the next run's
    if (!pb) {
      GS_CK(cudaMemcpy(&ctx->box, ctx->dbox.p, sizeof(GsBox), cudaMemcpyDeviceToHost));
      ctx->pbox = ctx->box;
      ctx->pbox_valid = true;
      ctx->pbox_gen++;
      ctx->pbox_d = d;
      ctx->pbox_dtype = in->dtype;
      ctx->pbox_h = cfg->h;
      ctx->pbox_w = ctx->img_w;
    } else {
      ctx->box = pbox_run;
    }
  }
  ctx->stats.slot_bytes = ctx->box.vol_frame <= 65536 ? 2 : 4;
  ctx->stats.predicted_box = pb ? 1 : 0;
  // ---- results
  if (ctx->hist_m.size() != (size_t)(rec ? nf : 0)) {
    ctx->hist_m.assign(rec ? nf : 0, {});
    ctx->hist_d.assign(rec ? nf : 0, {});
  }
  ctx->h_ffirst.assign(rb.fout, rb.fout + nf);
  ctx->h_k.assign(nf, 0);
  ctx->h_iters.assign(rb.fiters, rb.fiters + nf);
  ctx->h_conv.assign(rb.fconv, rb.fconv + nf);
  int64_t ktot = 0;
  for (int64_t f = 0; f < nf; ++f) {
    ctx->h_k[f] = rb.fk[f];
    ktot += rb.fk[f];
    out->k[f] = rb.fk[f];
    out->iterations[f] = rb.fiters[f];
    out->converged[f] = rb.fconv[f];
    swept += rb.fswept[f];
    if (rec)
      for (int t = g_iters[f]; t < rb.fiters[f]; ++t) {
        ctx->hist_m[f].push_back(rb.hm[(size_t)f * cfg->max_iter + t]);
        ctx->hist_d[f].push_back(rb.hd[(size_t)f * cfg->max_iter + t]);
      }
  }
  ctx->k_total = ktot;
  ctx->nframes = nf;
  ctx->have_run = true;
  gs_stats& s = ctx->stats;
  ctx->stats_times_pending = true;  // phase times are read from the events on demand
  s.cells_swept = swept;
  s.m0 = rb.ctr[0];
  s.k_total = ktot;
  s.max_iterations = 0;
  for (int64_t f = 0; f < nf; ++f) s.max_iterations = std::max(s.max_iterations, ctx->h_iters[f]);
  for (int k = 0; k < 3; ++k) s.sweep_modes[k] = rb.modes[k];
  for (int k = 0; k < 8; ++k) s.resident_cycles[k] = rb.modes[4 + k];
  s.fixed_shift = gs_fixed_shift(n, cfg->h);
  s.dense_cells = ctx->box.vol_total;
  hp.lap(3);
  return GS_OK;
}


// ---- frame-group pipeline for host-resident batches (e2e path of gs_run) ----
// Frames are independent, so a host batch is clustered as consecutive groups of
// frames: while group g runs on the engine stream, the copy stream stages group g+1 into the
// other staging buffer, and K7 of group g writes its labels straight into the caller's pinned
// memory (device->host, the other PCIe direction).  Each group is a complete engine run, so
// the results are exactly those of one whole-batch run; the centroids of every frame are
// collected on the host as the groups finish.
constexpr size_t kPipelineMinBytes = size_t(64) << 20;
constexpr size_t kPipelineGroupBytes = size_t(48) << 20;

bool want_pipeline(const gs_input* in, const gs_config* cfg) {
  if (in->on_device || in->batch < 2 || (cfg->flags & GS_NO_PIPELINE)) return false;
  if (cfg->flags & GS_DEBUG_PIPELINE) return true;
  return in->batch >= 4 && input_bytes(in) >= kPipelineMinBytes;
}

// frames per group: the largest divisor of nf whose group stays under the byte target (equal
// groups keep every group on the cached-shape path), at least 2 groups
int64_t group_frames(const gs_input* in, const gs_config* cfg) {
  const int64_t nf = in->batch;
  if (cfg->flags & GS_DEBUG_PIPELINE) return std::min<int64_t>(2, nf);
  const size_t fb = input_bytes(in) / (size_t)nf;
  int64_t cap = std::max<int64_t>(1, (int64_t)(kPipelineGroupBytes / std::max<size_t>(fb, 1)));
  cap = std::min<int64_t>(cap, nf / 2);
  for (int64_t g = cap; g >= std::max<int64_t>(1, cap / 2); --g)
    if (nf % g == 0) return g;
  return cap;
}

gs_status run_grouped(gs_ctx* ctx, const gs_input* in, const gs_config* cfg, gs_result* out) {
  const int64_t nf = in->batch, n = in->n, gf = group_frames(in, cfg);
  // group schedule: a short first group (the pipeline fill: its copy is not overlapped), then
  // groups of gf frames, the remainder last (three group shapes at most: the shape cache keeps
  // every group on the optimistic path)
  std::vector<int64_t> g0s, gcs;
  {
    int64_t f = 0;
    const int64_t first = (cfg->flags & GS_DEBUG_PIPELINE) ? gf : std::max<int64_t>(1, gf / 4);
    while (f < nf) {
      const int64_t c = std::min(f == 0 ? first : gf, nf - f);
      g0s.push_back(f);
      gcs.push_back(c);
      f += c;
    }
  }
  const int64_t G = (int64_t)g0s.size();
  const size_t fb = input_bytes(in) / (size_t)nf;
  const int d = in->d;
  cudaStream_t st = ctx->stream;
  if (!ctx->copy_stream) {
    GS_CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->ev_copy) GS_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  for (auto& b : ctx->stage) GS_TRY(grow(ctx, b, fb * (size_t)gf));
  // Pinned caller labels: K7 writes a group's labels to a device staging buffer at HBM speed
  // and the copy engine moves them out on a third stream while later groups are copied in and
  // run (zero-copy label stores from the SMs made K7 itself PCIe-bound and slowed the
  // concurrent input copies); pageable labels keep the in-stream copy of run_impl.
  const bool dma_out = !(cfg->flags & GS_DEVICE_OUTPUTS) && graph_safe(out->labels);
  if (dma_out) {
    if (!ctx->d2h_stream) {
      GS_CK(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
      for (auto& e : ctx->ev_d2h) GS_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    for (auto& b : ctx->lab_stage) GS_TRY(grow(ctx, b, sizeof(int32_t) * (size_t)n * (size_t)gf));
  }
  const char* src = static_cast<const char*>(in->points);
  auto stage_in = [&](int64_t g) -> gs_status {
    const int64_t f0 = g0s[g], cnt = gcs[g];
    GS_CK(cudaMemcpyAsync(ctx->stage[g & 1].p, src + (size_t)f0 * fb, fb * (size_t)cnt,
                          cudaMemcpyHostToDevice, ctx->copy_stream));
    GS_CK(cudaEventRecord(ctx->ev_copy[g & 1], ctx->copy_stream));
    return GS_OK;
  };
  std::vector<double> cent;
  std::vector<int64_t> off(nf + 1, 0);
  std::vector<int64_t> all_k(nf);
  std::vector<int32_t> all_it(nf), all_cv(nf);
  std::vector<std::vector<int64_t>> hm;
  std::vector<std::vector<double>> hd;
  const bool rec = (cfg->flags & GS_RECORD_HISTORY) != 0;
  if (rec) {
    hm.resize(nf);
    hd.resize(nf);
  }
  gs_stats agg{};
  const bool graphs = ctx->use_graphs;
  ctx->use_graphs = false;  // the buffers change every group: plain launches, no re-capture
  gs_status s = stage_in(0);
  int64_t f0 = 0;
  for (int64_t g = 0; g < G && s == GS_OK; ++g) {
    f0 = g0s[g];
    const int64_t cnt = gcs[g];
    // the other staging buffer was last read by group g-1, which has completed (synchronous)
    if (g + 1 < G && (s = stage_in(g + 1)) != GS_OK) break;
    if (cudaStreamWaitEvent(st, ctx->ev_copy[g & 1], 0) != cudaSuccess) {
      s = fail(ctx, GS_E_CUDA, "cudaStreamWaitEvent");
      break;
    }
    gs_input sub = *in;
    sub.points = ctx->stage[g & 1].p;
    sub.batch = cnt;
    sub.on_device = 1;
    gs_result r{out->labels + (size_t)f0 * n, out->k + f0, out->iterations + f0,
                out->converged + f0};
    gs_config c = *cfg;
    c.flags &= ~(uint32_t)(GS_DEBUG_PIPELINE | GS_DEVICE_OUTPUTS);
    if (dma_out) {
      // the staging buffer was last drained by group g-2's copy
      if (g >= 2 && cudaStreamWaitEvent(st, ctx->ev_d2h[g & 1], 0) != cudaSuccess) {
        s = fail(ctx, GS_E_CUDA, "cudaStreamWaitEvent");
        break;
      }
      r.labels = ctx->lab_stage[g & 1].as<int32_t>();
      c.flags |= GS_DEVICE_OUTPUTS;
    }
    if ((s = run_impl(ctx, &sub, &c, &r)) != GS_OK) {
      ctx->err = "frames " + std::to_string((long long)f0) + "-" +
                 std::to_string((long long)(f0 + cnt - 1)) + ": " + ctx->err;
      break;
    }
    if (dma_out) {  // (run_impl has synchronised: the group's labels are in the staging buffer)
      if (cudaMemcpyAsync(out->labels + (size_t)f0 * n, ctx->lab_stage[g & 1].p,
                          sizeof(int32_t) * (size_t)n * (size_t)cnt, cudaMemcpyDeviceToHost,
                          ctx->d2h_stream) != cudaSuccess ||
          cudaEventRecord(ctx->ev_d2h[g & 1], ctx->d2h_stream) != cudaSuccess) {
        s = fail(ctx, GS_E_CUDA, "label copy");
        break;
      }
    }
    // this group's centroids (rows h_ffirst[f] .. + h_k[f] of the final cell buffer)
    int64_t lo = INT64_MAX, hi = 0;
    for (int64_t f = 0; f < cnt; ++f) {
      lo = std::min<int64_t>(lo, ctx->h_ffirst[f]);
      hi = std::max<int64_t>(hi, ctx->h_ffirst[f] + ctx->h_k[f]);
    }
    std::vector<double> rows((size_t)std::max<int64_t>(hi - lo, 0) * d);
    if (hi > lo &&
        cudaMemcpy(rows.data(), ctx->S[ctx->cur].as<double>() + (size_t)lo * d,
                   sizeof(double) * rows.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      s = fail(ctx, GS_E_CUDA, "centroid readback");
      break;
    }
    for (int64_t f = 0; f < cnt; ++f) {
      const int64_t k = ctx->h_k[f];
      off[f0 + f] = (int64_t)(cent.size() / d);
      const double* r0 = rows.data() + (size_t)(ctx->h_ffirst[f] - lo) * d;
      cent.insert(cent.end(), r0, r0 + (size_t)k * d);
      all_k[f0 + f] = k;
      all_it[f0 + f] = ctx->h_iters[f];
      all_cv[f0 + f] = ctx->h_conv[f];
      if (rec) {
        hm[f0 + f] = ctx->hist_m[f];
        hd[f0 + f] = ctx->hist_d[f];
      }
    }
    const gs_stats& gs1 = ctx->stats;
    agg.cells_swept += gs1.cells_swept;
    agg.m0 += gs1.m0;
    agg.k_total += gs1.k_total;
    agg.kernel_launches += gs1.kernel_launches;
    agg.lib_calls += gs1.lib_calls;
    agg.max_iterations = std::max(agg.max_iterations, gs1.max_iterations);
    agg.fixed_shift = gs1.fixed_shift;
    agg.dense_cells = std::max(agg.dense_cells, gs1.dense_cells);
    for (int k = 0; k < 3; ++k) agg.sweep_modes[k] += gs1.sweep_modes[k];
    for (int k = 0; k < 8; ++k) agg.resident_cycles[k] += gs1.resident_cycles[k];
  }
  ctx->use_graphs = graphs;
  cudaStreamSynchronize(ctx->copy_stream);  // no staging copy outlives the call
  if (ctx->d2h_stream && cudaStreamSynchronize(ctx->d2h_stream) != cudaSuccess && s == GS_OK)
    s = fail(ctx, GS_E_CUDA, "label copy");
  if (s != GS_OK) {
    ctx->have_run = false;
    ctx->grouped = false;
    return s;
  }
  off[nf] = (int64_t)(cent.size() / d);
  ctx->g_cent.swap(cent);
  ctx->g_cent_off.swap(off);
  ctx->grouped = true;
  ctx->group_f0 = f0;
  ctx->nframes = nf;
  ctx->h_k = all_k;
  ctx->h_iters = all_it;
  ctx->h_conv = all_cv;
  if (rec) {
    ctx->hist_m.swap(hm);
    ctx->hist_d.swap(hd);
  }
  ctx->k_total = agg.k_total;
  ctx->stats = agg;  // phase times: those of the last group's events
  ctx->have_run = true;
  return GS_OK;
}

// ---- MS++ baseline (gs_mspp.cuh) ----
template <int D, typename T>
gs_status mspp_launch(gs_ctx* ctx, const void* dpts, int64_t n, int64_t m0, double tol,
                      int32_t max_iter, int MS, int vol_small, double* snew0,
                      unsigned long long* disp0, int* outw, double* dhist, double* cent) {
  cudaStream_t st = ctx->stream;
  gs::k_mspp_jacobi<D><<<blocks_for(m0, 128), 128, 0, st>>>(
      (int)m0, ctx->dbox.as<GsBox>(), ctx->ckey[0].as<uint32_t>(), ctx->ccnt[0].as<uint32_t>(),
      ctx->S[0].as<double>(), ctx->idx.as<int32_t>(), snew0);
  GS_LAUNCHED("k_mspp_jacobi");
  gs::k_mspp_disp0<D, T><<<blocks_for(n, 256, (int64_t)ctx->num_sms * 8), 256, 0, st>>>(
      n, (const T*)dpts, ctx->slot.p, ctx->dbox.as<GsBox>(), ctx->idx.as<int32_t>(), snew0, disp0);
  GS_LAUNCHED("k_mspp_disp0");
  if (m0 > MS) {  // ---- the first grid exceeds one CTA: later iterations on all SMs
    const int64_t V = ctx->box.vol_total;
    GS_TRY(grow(ctx, ctx->mpos, sizeof(double) * (size_t)m0 * D));
    GS_TRY(grow(ctx, ctx->mpc, sizeof(uint32_t) * (size_t)m0));
    GS_TRY(grow(ctx, ctx->mkey, sizeof(uint32_t) * (size_t)m0));
    GS_TRY(grow(ctx, ctx->mroot, sizeof(int32_t) * (size_t)m0));
    GS_TRY(grow(ctx, ctx->msnew, sizeof(double) * (size_t)m0 * D));
    unsigned* cnt32 = ctx->counters.as<unsigned>();
    // particles = the initial cells at iteration 0's positions; the first grid's index released
    GS_CK(cudaMemcpyAsync(ctx->mpos.p, snew0, sizeof(double) * (size_t)m0 * D,
                          cudaMemcpyDeviceToDevice, st));
    GS_CK(cudaMemcpyAsync(ctx->mpc.p, ctx->ccnt[0].p, sizeof(uint32_t) * (size_t)m0,
                          cudaMemcpyDeviceToDevice, st));
    gs::k_iota<<<blocks_for(m0, 256), 256, 0, st>>>((int)m0, ctx->mroot.as<int32_t>());
    GS_LAUNCHED("k_iota");
    gs::k_idx_clear<<<blocks_for(m0, 256), 256, 0, st>>>((int)m0, ctx->ckey[0].as<uint32_t>(),
                                                          ctx->idx.as<int32_t>());
    GS_LAUNCHED("k_idx_clear");
    std::vector<double> hd((size_t)max_iter, 0.0);
    unsigned long long d0b = 0;
    GS_CK(cudaMemcpyAsync(&d0b, disp0, 8, cudaMemcpyDeviceToHost, st));
    GS_CK(cudaStreamSynchronize(st));
    double dsp;
    std::memcpy(&dsp, &d0b, 8);
    hd[0] = dsp;
    int it = 1;
    bool conv = dsp < tol;
    bool final_pass = conv || it >= max_iter;
    int64_t mp = m0;
    const unsigned tg = (unsigned)std::min<int64_t>(V / gs::kOccTile + 1, (int64_t)ctx->num_sms * 4);
    unsigned long long* dmax = disp0;  // reused: the displacement of the current iteration
    for (;;) {
      // re-grid the particles (pins M1, M4)
      gs::k_mspp_bin_g<D><<<blocks_for(mp, 256), 256, 0, st>>>(
          (int)mp, ctx->mpos.as<double>(), ctx->mpc.as<uint32_t>(), ctx->dbox.as<GsBox>(),
          ctx->box.scale, ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>(),
          ctx->mkey.as<uint32_t>(), ctx->epoch_dev.as<unsigned>(), cnt32 + 5,
          ctx->errflag.as<int>());
      GS_LAUNCHED("k_mspp_bin_g");
      gs::k_occ<<<tg, 256, 0, st>>>(
          ctx->dbox.as<GsBox>(), ctx->epoch_dev.as<unsigned>(), ctx->tiles.as<unsigned long long>(),
          cnt32 + 5, cnt32, ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>(),
          ctx->ckey[1].as<uint32_t>(), ctx->ccnt[1].as<uint32_t>(), ctx->S[1].as<double>(),
          ctx->idx.as<int32_t>(), ctx->root.as<int32_t>(), ctx->initkey.as<uint32_t>(),
          ctx->ifirst.as<int32_t>(), ctx->errflag.as<int>());
      GS_LAUNCHED("k_occ");
      if (final_pass) {  // pin M5: the final cells, ids = lex ranks
        gs::k_mspp_root_g<<<blocks_for(m0, 256), 256, 0, st>>>(
            (int)m0, ctx->mroot.as<int32_t>(), ctx->mkey.as<uint32_t>(), ctx->idx.as<int32_t>(),
            ctx->ckey[0].as<uint32_t>(), ctx->lab.as<int32_t>());
        GS_LAUNCHED("k_mspp_root_g");
        unsigned mfin = 0;
        GS_CK(cudaMemcpyAsync(&mfin, cnt32, 4, cudaMemcpyDeviceToHost, st));
        GS_CK(cudaStreamSynchronize(st));
        gs::k_idx_clear<<<blocks_for(mfin, 256), 256, 0, st>>>(
            (int)mfin, ctx->ckey[1].as<uint32_t>(), ctx->idx.as<int32_t>());
        GS_LAUNCHED("k_idx_clear");
        const int ow[4] = {(int)mfin, it, conv ? 1 : 0, 0};
        GS_CK(cudaMemcpyAsync(outw, ow, sizeof(ow), cudaMemcpyHostToDevice, st));
        if (dhist)
          GS_CK(cudaMemcpyAsync(dhist, hd.data(), sizeof(double) * hd.size(),
                                cudaMemcpyHostToDevice, st));
        GS_CK(cudaStreamSynchronize(st));  // (hd and ow are host stack memory)
        return GS_OK;
      }
      // update (pin M2), displacement (M3), particle -> cell of the initial roots (M4)
      GS_CK(cudaMemsetAsync(dmax, 0, 8, st));
      gs::k_mspp_jacobi_g<D><<<blocks_for(mp, 128), 128, 0, st>>>(
          cnt32, ctx->dbox.as<GsBox>(), ctx->ckey[1].as<uint32_t>(), ctx->ccnt[1].as<uint32_t>(),
          ctx->S[1].as<double>(), ctx->idx.as<int32_t>(), ctx->msnew.as<double>());
      GS_LAUNCHED("k_mspp_jacobi_g");
      gs::k_mspp_disp_g<D><<<blocks_for(mp, 256), 256, 0, st>>>(
          (int)mp, ctx->mpos.as<double>(), ctx->mkey.as<uint32_t>(), ctx->idx.as<int32_t>(),
          ctx->msnew.as<double>(), dmax);
      GS_LAUNCHED("k_mspp_disp_g");
      gs::k_mspp_root_g<<<blocks_for(m0, 256), 256, 0, st>>>(
          (int)m0, ctx->mroot.as<int32_t>(), ctx->mkey.as<uint32_t>(), ctx->idx.as<int32_t>(),
          nullptr, nullptr);
      GS_LAUNCHED("k_mspp_root_g");
      gs::k_mspp_next_g<D><<<blocks_for(mp, 256), 256, 0, st>>>(
          cnt32, ctx->msnew.as<double>(), ctx->ccnt[1].as<uint32_t>(), ctx->ckey[1].as<uint32_t>(),
          ctx->mpos.as<double>(), ctx->mpc.as<uint32_t>(), ctx->idx.as<int32_t>());
      GS_LAUNCHED("k_mspp_next_g");
      unsigned long long rb[2] = {0, 0};
      GS_CK(cudaMemcpyAsync(&rb[0], dmax, 8, cudaMemcpyDeviceToHost, st));
      GS_CK(cudaMemcpyAsync(&rb[1], cnt32, 4, cudaMemcpyDeviceToHost, st));
      GS_CK(cudaStreamSynchronize(st));
      int err = 0;
      GS_CK(cudaMemcpy(&err, ctx->errflag.p, sizeof(int), cudaMemcpyDeviceToHost));
      if (err & 2) return fail(ctx, GS_E_INTERNAL_INVARIANT, "an MS++ particle left the key box");
      std::memcpy(&dsp, &rb[0], 8);
      mp = (int64_t)(unsigned)rb[1];
      hd[(size_t)it] = dsp;
      ++it;
      conv = dsp < tol;
      final_pass = conv || it >= max_iter;
    }
  }
  gs::MsppArgs a;
  a.m0 = (int)m0;
  a.MS = MS;
  a.F = ctx->box.F;
  a.max_iter = max_iter;
  a.vol_small = vol_small;
  a.tol = tol;
  a.scale = ctx->box.scale;
  a.inv_scale = ctx->box.inv_scale;
  a.pb = ctx->dbox.as<GsBox>();
  a.ckey0 = ctx->ckey[0].as<uint32_t>();
  a.ccnt0 = ctx->ccnt[0].as<uint32_t>();
  a.Snew0 = snew0;
  a.idx = ctx->idx.as<int32_t>();
  a.lab = ctx->lab.as<int32_t>();
  a.disp0 = disp0;
  a.cent_out = cent;
  a.out = outw;
  a.disp_hist = dhist;
  const size_t smem = (size_t)MS * gs::mspp_bytes_per_slot<D>() +
                      (vol_small ? 2 * (size_t)ctx->box.vol_frame : 0);
  GS_CK(cudaFuncSetAttribute(gs::k_mspp_loop<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem));
  gs::k_mspp_loop<D><<<1, 512, smem, st>>>(a);
  GS_LAUNCHED("k_mspp_loop");
  return GS_OK;
}

}  // namespace

extern "C" gs_status gs_mspp_run(gs_ctx* ctx, const gs_input* in, double h, double tol,
                                 int32_t max_iter, gs_result* out, double* disp_hist) {
  gs_config cfg{h, max_iter, 0};
  gs_status s0 = validate(in, &cfg);
  if (s0 != GS_OK) {
    if (ctx) ctx->err = gs_status_string(s0);
    return s0;
  }
  if (!ctx || !out || !out->labels || !out->k || !out->iterations || !out->converged)
    return GS_E_INVALID_PARAMETER;
  ctx->err.clear();
  if (in->batch != 1) return fail(ctx, GS_E_INVALID_PARAMETER, "MS++ runs one dataset (batch 1)");
  if (in->dtype != GS_F32 && in->dtype != GS_F64)
    return fail(ctx, GS_E_INVALID_PARAMETER, "MS++ takes fp32/fp64 features");
  if (in->d > 6) return fail(ctx, GS_E_INVALID_PARAMETER, "MS++ baseline: d <= 6");
  if (!(tol > 0.0) || !std::isfinite(tol))
    return fail(ctx, GS_E_INVALID_PARAMETER, "tol must be > 0 (SPEC.md:242)");
  cudaSetDevice(ctx->device);
  ctx->have_run = false;
  ctx->grouped = false;
  ctx->img_w = 0;
  ctx->stats = gs_stats{};  // (kernel_launches of this MS++ run)
  cudaGetLastError();
  const int d = in->d;
  const int64_t n = in->n;
  const void* dpts = in->points;
  if (!in->on_device) {
    GS_TRY(grow(ctx, ctx->pts, input_bytes(in)));
    GS_CK(cudaMemcpyAsync(ctx->pts.p, in->points, input_bytes(in), cudaMemcpyHostToDevice,
                          ctx->stream));
    dpts = ctx->pts.p;
  }
  GS_TRY(grow(ctx, ctx->errflag, 32));
  GS_TRY(grow(ctx, ctx->counters, 64));
  GS_TRY(ensure_frames(ctx, 1));
  int64_t m0 = 0;
  for (int attempt = 0;; ++attempt) {  // the first grid (pin M1) = the engine's n-scale phase
    GS_TRY(launch_nscale(ctx, dpts, in->dtype, d, n, 1, h));
    int hdr[8];
    unsigned ctr[16];
    GS_CK(cudaMemcpyAsync(hdr, ctx->errflag.p, 32, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CK(cudaMemcpyAsync(ctr, ctx->counters.p, 64, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CK(cudaMemcpyAsync(&ctx->box, ctx->dbox.p, sizeof(GsBox), cudaMemcpyDeviceToHost,
                          ctx->stream));
    GS_CK(cudaStreamSynchronize(ctx->stream));
    if ((hdr[0] & 32) && attempt < 3) {
      GS_TRY(grow_dense_for(ctx, *(long long*)(hdr + 2), d));
      continue;
    }
    if (hdr[0] & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
    if (hdr[0] & (32 | 64)) return fail(ctx, GS_E_KEY_RANGE, "key box too large");
    m0 = ctr[0];
    break;
  }
  ctx->ctl_clean = false;
  // one CTA holds the particles: the largest power-of-two slot count that fits with the
  // frame's dense index (in shared memory when it fits, else the global grid index)
  const size_t budget = 226 * 1024;
  const size_t bps = (size_t)(d == 1 ? gs::mspp_bytes_per_slot<1>() : d == 2 ? gs::mspp_bytes_per_slot<2>()
                              : d == 3 ? gs::mspp_bytes_per_slot<3>() : d == 4 ? gs::mspp_bytes_per_slot<4>()
                              : d == 5 ? gs::mspp_bytes_per_slot<5>() : gs::mspp_bytes_per_slot<6>());
  int MS = 1;
  while ((size_t)(2 * MS) * bps <= budget) MS *= 2;
  int vol_small = 0;
  if (2 * (size_t)ctx->box.vol_frame + (size_t)MS * bps <= budget) vol_small = 1;
  else if (2 * (size_t)ctx->box.vol_frame + (size_t)(MS / 2) * bps <= budget && m0 <= MS / 2) {
    MS /= 2;
    vol_small = 1;
  }
  GS_TRY(grow(ctx, ctx->S1, sizeof(double) * (size_t)m0 * d));
  GS_TRY(ensure_cells(ctx, m0, d));  // (the all-SM loop re-grids into the second cell buffers)
  GS_TRY(grow(ctx, ctx->dbg, 64 + sizeof(double) * (size_t)max_iter));
  GS_CK(cudaMemsetAsync(ctx->dbg.p, 0, 64, ctx->stream));
  unsigned long long* disp0 = (unsigned long long*)ctx->dbg.p;
  int* outw = (int*)((char*)ctx->dbg.p + 16);
  double* dhist = (double*)((char*)ctx->dbg.p + 64);
  double* cent = ctx->S[1].as<double>();
  double* snew0 = ctx->S1.as<double>();
  gs_status ls = GS_OK;
  const bool f64 = in->dtype == GS_F64;
  switch (d) {
#define GS_CASE(D)                                                                              \
  case D:                                                                                       \
    ls = f64 ? mspp_launch<D, double>(ctx, dpts, n, m0, tol, max_iter, MS, vol_small, snew0,   \
                                      disp0, outw, dhist, cent)                                 \
             : mspp_launch<D, float>(ctx, dpts, n, m0, tol, max_iter, MS, vol_small, snew0,    \
                                     disp0, outw, dhist, cent);                                 \
    break;
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
#undef GS_CASE
  }
  GS_TRY(ls);
  GS_TRY(grow(ctx, ctx->labels, sizeof(int32_t) * n));
  int32_t* dl = ctx->labels.as<int32_t>();
  gs::k_label<false><<<label_grid(ctx, n, 1), 256, 0, ctx->stream>>>(
      n, 1, ctx->slot.p, ctx->dbox.as<GsBox>(), ctx->lab.as<int32_t>(), dl, nullptr, nullptr, 0,
      0);
  GS_LAUNCHED("k_label");
  GS_CK(cudaMemcpyAsync(out->labels, dl, sizeof(int32_t) * n, cudaMemcpyDeviceToHost,
                        ctx->stream));
  int ow[4];
  GS_CK(cudaMemcpyAsync(ow, outw, sizeof(ow), cudaMemcpyDeviceToHost, ctx->stream));
  if (disp_hist)
    GS_CK(cudaMemcpyAsync(disp_hist, dhist, sizeof(double) * max_iter, cudaMemcpyDeviceToHost,
                          ctx->stream));
  int err = 0;
  GS_CK(cudaMemcpyAsync(&err, ctx->errflag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaStreamSynchronize(ctx->stream));
  GS_CK(cudaGetLastError());
  if (err & ~0) {
    if (err & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
    if (err & 2) return fail(ctx, GS_E_INTERNAL_INVARIANT, "a point's key left the box");
  }
  out->k[0] = ow[0];
  out->iterations[0] = ow[1];
  out->converged[0] = ow[2];
  ctx->cur = 1;  // gs_get_centroids reads the final centroids from S[1]
  ctx->nframes = 1;
  ctx->h_k.assign(1, ow[0]);
  ctx->h_ffirst.assign(1, 0);
  ctx->hist_m.clear();
  ctx->hist_d.clear();
  ctx->have_run = true;
  return GS_OK;
}

namespace {
}  // namespace

extern "C" {

int32_t gs_fixed_shift(int64_t n, double h) {
  // mirrors oracle fixed_shift(): |sum| < 2^61 for any cell of <= n points, offsets in [~0, h]
  int ln = 0;
  while ((int64_t(1) << ln) < n) ++ln;
  int eh = std::ilogb(h) + 1;
  int F = 61 - ln - eh;
  return std::max(-1000, std::min(1000, F));
}

const char* gs_status_string(gs_status s) {
  switch (s) {
    case GS_OK: return "ok";
    case GS_E_INVALID_INPUT: return "invalid input";
    case GS_E_INVALID_BANDWIDTH: return "invalid bandwidth";
    case GS_E_EMPTY_INPUT: return "empty input";
    case GS_E_INVALID_PARAMETER: return "invalid parameter";
    case GS_E_INTERNAL_INVARIANT: return "internal invariant violated";
    case GS_E_KEY_RANGE: return "key range exceeds the dense cell grid";
    case GS_E_TUNING_FAILED: return "tuning failure";
    case GS_E_UNDEFINED_SCORE: return "undefined score";
    case GS_E_INVALID_WINDOW: return "invalid window";
    case GS_E_SELECTION: return "selection error";
    case GS_E_CUDA: return "CUDA error";
    case GS_E_OOM: return "device out of memory";
    case GS_E_NCCL: return "NCCL error";
    case GS_E_NO_DEVICE: return "no CUDA device";
  }
  return "unknown status";
}

gs_status gs_validate(const gs_input* in, const gs_config* cfg) { return validate(in, cfg); }

gs_status gs_create(int device, void* cuda_stream, gs_ctx** out) {
  if (!out) return GS_E_INVALID_PARAMETER;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device || device < 0) {
    cudaGetLastError();
    return GS_E_NO_DEVICE;
  }
  gs_ctx* ctx = new gs_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return GS_E_NO_DEVICE;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return GS_E_CUDA;
    }
    ctx->own_stream = true;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  *out = ctx;
  return GS_OK;
}

void gs_destroy(gs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (DevBuf* b : {&ctx->cnt, &ctx->qs, &ctx->idx, &ctx->lab, &ctx->pts, &ctx->slot,
                    &ctx->labels, &ctx->occ, &ctx->occ_sorted, &ctx->ckey[0], &ctx->ckey[1],
                    &ctx->ccnt[0], &ctx->ccnt[1], &ctx->S[0], &ctx->S[1], &ctx->S1, &ctx->nbl,
                    &ctx->nbn, &ctx->nbe, &ctx->den, &ctx->flag, &ctx->nkey, &ctx->vals,
                    &ctx->skey, &ctx->sval, &ctx->head, &ctx->sid, &ctx->segstart, &ctx->parent,
                    &ctx->root, &ctx->initkey, &ctx->fdone, &ctx->fchanged, &ctx->fadj,
                    &ctx->fm, &ctx->fdisp, &ctx->ffirst, &ctx->fcount, &ctx->ifirst, &ctx->icount,
                    &ctx->fiters, &ctx->fconv, &ctx->fk, &ctx->hist, &ctx->counters, &ctx->errflag,
                    &ctx->bpart, &ctx->cub_tmp, &ctx->dbg, &ctx->modes, &ctx->tiles,
                    &ctx->dbox, &ctx->erec, &ctx->lprod, &ctx->rden, &ctx->lvl,
                    &ctx->lsucc, &ctx->order, &ctx->xsum, &ctx->pkeys, &ctx->pcounts,
                    &ctx->psums, &ctx->npend, &ctx->epoch_dev, &ctx->fswept, &ctx->fout, &ctx->ctl})
    b->release();
  for (auto& b : ctx->stage) b.release();
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  for (auto& e : ctx->ev_copy)
    if (e) cudaEventDestroy(e);
  if (ctx->d2h_stream) {
    cudaStreamSynchronize(ctx->d2h_stream);
    cudaStreamDestroy(ctx->d2h_stream);
  }
  for (auto& e : ctx->ev_d2h)
    if (e) cudaEventDestroy(e);
  for (auto& b : ctx->lab_stage) b.release();
  if (ctx->pin) cudaFreeHost(ctx->pin);
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  if (ctx->ev_plan) cudaEventDestroy(ctx->ev_plan);
  ctx->iterpack.release();
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* gs_last_error(const gs_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

gs_status gs_run(gs_ctx* ctx, const gs_input* in, const gs_config* cfg, gs_result* out) {
  gs_status s = validate(in, cfg);
  if (s != GS_OK) {
    if (ctx) ctx->err = gs_status_string(s);
    return s;
  }
  if (!ctx) return GS_E_INVALID_PARAMETER;
  ctx->err.clear();
  if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GS_E_CUDA, "cudaSetDevice");
  ctx->grouped = false;
  if (want_pipeline(in, cfg)) {
    if (!out || !out->labels || !out->k || !out->iterations || !out->converged)
      return fail(ctx, GS_E_INVALID_PARAMETER, "null result buffer");
    return run_grouped(ctx, in, cfg, out);
  }
  return run_impl(ctx, in, cfg, out);
}

gs_status gs_get_centroids(gs_ctx* ctx, int64_t frame, double* out, int64_t cap_k) {
  if (!ctx || !out) return GS_E_INVALID_PARAMETER;
  if (!ctx->have_run || frame < 0 || frame >= ctx->nframes)
    return fail(ctx, GS_E_INVALID_PARAMETER, "no such frame in the last run");
  const int64_t k = ctx->h_k[frame];
  if (cap_k < k) return fail(ctx, GS_E_INVALID_PARAMETER, "centroid buffer too small");
  const int d = ctx->box.d;
  if (ctx->grouped) {  // pipelined run: collected on the host as the groups finished
    std::memcpy(out, ctx->g_cent.data() + (size_t)ctx->g_cent_off[frame] * d,
                sizeof(double) * k * d);
    return GS_OK;
  }
  GS_CK(cudaMemcpyAsync(out, ctx->S[ctx->cur].as<double>() + (size_t)ctx->h_ffirst[frame] * d,
                        sizeof(double) * k * d, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaStreamSynchronize(ctx->stream));
  return GS_OK;
}

gs_status gs_get_history(gs_ctx* ctx, int64_t frame, int64_t* m_t, double* maxdisp_t,
                         int32_t cap) {
  if (!ctx) return GS_E_INVALID_PARAMETER;
  if (!ctx->have_run || frame < 0 || frame >= (int64_t)ctx->hist_m.size())
    return fail(ctx, GS_E_INVALID_PARAMETER, "no history for this frame (GS_RECORD_HISTORY?)");
  const auto& hm = ctx->hist_m[frame];
  const auto& hd = ctx->hist_d[frame];
  for (int32_t t = 0; t < cap && t < (int32_t)hm.size(); ++t) {
    if (m_t) m_t[t] = hm[t];
    if (maxdisp_t) maxdisp_t[t] = hd[t];
  }
  return GS_OK;
}

gs_status gs_get_stats(gs_ctx* ctx, gs_stats* out) {
  if (!ctx || !out) return GS_E_INVALID_PARAMETER;
  if (ctx->stats_times_pending) {  // the last run's phase events (all complete: it synced)
    ctx->stats_times_pending = false;
    cudaSetDevice(ctx->device);
    gs_stats& s = ctx->stats;
    auto el = [&](int a, int b) {
      float ms = 0;
      if (((ctx->ev_mask >> a) & 1u) && ((ctx->ev_mask >> b) & 1u))
        cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]);
      return (double)ms;
    };
    s.ms_h2d = el(0, 1);
    s.ms_bin = el(1, 2);
    s.ms_iterate = el(2, 3);
    s.ms_label = el(3, 4);
    s.ms_d2h = el(4, 5);
    s.ms_total = el(1, 4);
    s.ms_k_bin = el(6, 7);
    s.ms_k_label = el(3, 4);
    cudaGetLastError();  // timing is best-effort diagnostics
  }
  *out = ctx->stats;
  return GS_OK;
}

gs_status gs_shard_keybounds(gs_ctx* ctx, const gs_input* in, double h, int64_t* klo,
                             int64_t* khi) {
  gs_config cfg{h, 1, 0};
  gs_status s = validate(in, &cfg);
  if (s != GS_OK) return s;
  if (!ctx || !klo || !khi) return GS_E_INVALID_PARAMETER;
  if (in->batch != 1) return fail(ctx, GS_E_INVALID_PARAMETER, "a shard is one frame");
  if (img_width(in)) return fail(ctx, GS_E_INVALID_PARAMETER, "rgbxy pixels cannot be sharded");
  ctx->err.clear();
  ctx->img_w = 0;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const int d = in->d;
  const int64_t n = in->n;
  const void* dpts = in->points;
  if (!in->on_device) {
    GS_TRY(grow(ctx, ctx->pts, input_bytes(in)));
    GS_CK(cudaMemcpyAsync(ctx->pts.p, in->points, input_bytes(in), cudaMemcpyHostToDevice, st));
    dpts = ctx->pts.p;
  }
  const unsigned nblk = blocks_for(n, 256 * 4, (int64_t)ctx->num_sms * 2);
  GS_TRY(grow(ctx, ctx->bpart, sizeof(double) * nblk * d * 2));
  GS_TRY(grow(ctx, ctx->dbox, sizeof(GsBox)));
  GS_TRY(ensure_frames(ctx, 1));
  if (!ctx->epoch_dev.p) {
    GS_TRY(grow(ctx, ctx->epoch_dev, 16));
    GS_CK(cudaMemsetAsync(ctx->epoch_dev.p, 0, 16, st));
  }
  GS_CK(cudaMemsetAsync(ctx->ctl.p, 0, ctl_zero_bytes(ctx->ctl_nf), st));
  ctx->ctl_clean = false;
  GS_TRY(dispatch_bounds_bin(ctx, dpts, in->dtype, d, n, true, nblk, h, n, 1));
  int hdr[8];
  GsBox b;
  GS_CK(cudaMemcpyAsync(hdr, ctx->errflag.p, 32, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(&b, ctx->dbox.p, sizeof(GsBox), cudaMemcpyDeviceToHost, st));
  GS_CK(cudaStreamSynchronize(st));
  if (hdr[0] & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
  if (hdr[0] & 64) return fail(ctx, GS_E_KEY_RANGE, "cell keys exceed the int64 key range");
  for (int c = 0; c < d; ++c) {
    klo[c] = b.kmin[c] + GS_APRON;
    khi[c] = b.kmin[c] + b.ext[c] - 1 - GS_APRON;
  }
  ctx->ctl_clean = false;
  return GS_OK;
}

gs_status gs_shard_bin(gs_ctx* ctx, const gs_input* in, double h, int64_t n_global,
                       const int64_t* klo, const int64_t* khi, int64_t cap, int64_t* m_out,
                       uint32_t* keys, uint32_t* counts, int64_t* sums) {
  gs_config cfg{h, 1, 0};
  gs_status s = validate(in, &cfg);
  if (s != GS_OK) return s;
  if (!ctx || !klo || !khi || !m_out || (cap > 0 && (!keys || !counts || !sums)))
    return GS_E_INVALID_PARAMETER;
  if (in->batch != 1) return fail(ctx, GS_E_INVALID_PARAMETER, "a shard is one frame");
  if (n_global < in->n) return fail(ctx, GS_E_INVALID_PARAMETER, "n_global < shard size");
  if (img_width(in)) return fail(ctx, GS_E_INVALID_PARAMETER, "rgbxy pixels cannot be sharded");
  ctx->err.clear();
  ctx->img_w = 0;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const int d = in->d;
  const int64_t n = in->n;
  // the global box: same keys, strides and fixed-point exponent on every rank
  GsBox b;
  std::memset(&b, 0, sizeof(b));
  b.d = d;
  b.h = h;
  b.inv_h = 1.0 / h;  // == __drcp_rn(h): both correctly rounded
  b.F = gs_fixed_shift(n_global, h);
  b.scale = std::ldexp(1.0, b.F);
  b.inv_scale = std::ldexp(1.0, -b.F);
  b.n = n;
  b.nframes = 1;
  double vol = 1.0;
  for (int c = 0; c < d; ++c) {
    if (khi[c] < klo[c]) return fail(ctx, GS_E_INVALID_PARAMETER, "empty key range");
    b.kmin[c] = klo[c] - GS_APRON;
    b.ext[c] = khi[c] - klo[c] + 1 + 2 * GS_APRON;
    vol *= (double)b.ext[c];
  }
  if (vol > (double)kMaxDenseCells)
    return fail(ctx, GS_E_KEY_RANGE, "key box exceeds the dense cell grid (2^28)");
  int64_t sv = 1;
  for (int c = d - 1; c >= 0; --c) {
    b.stride[c] = sv;
    sv *= b.ext[c];
  }
  b.vol_frame = b.vol_total = sv;
  GS_TRY(ensure_dense(ctx, std::max<int64_t>(ctx->dense_cap, sv), d));
  GS_TRY(ensure_cells(ctx, std::min<int64_t>(n, sv), d));
  GS_TRY(ensure_frames(ctx, 1));
  GS_TRY(grow(ctx, ctx->slot, sizeof(uint32_t) * n));
  GS_TRY(grow(ctx, ctx->dbox, sizeof(GsBox)));
  GS_TRY(grow(ctx, ctx->xsum, 8 * (size_t)d * std::min<int64_t>(n, sv)));
  const int64_t ntiles = ctx->dense_cap / gs::kOccTile + 1;
  if (ctx->tiles.bytes < sizeof(unsigned long long) * ntiles) {
    GS_TRY(grow(ctx, ctx->tiles, sizeof(unsigned long long) * ntiles));
    GS_CK(cudaMemsetAsync(ctx->tiles.p, 0, ctx->tiles.bytes, st));
  }
  if (!ctx->epoch_dev.p) {
    GS_TRY(grow(ctx, ctx->epoch_dev, 16));
    GS_CK(cudaMemsetAsync(ctx->epoch_dev.p, 0, 16, st));
  }
  const void* dpts = in->points;
  if (!in->on_device) {
    GS_TRY(grow(ctx, ctx->pts, input_bytes(in)));
    GS_CK(cudaMemcpyAsync(ctx->pts.p, in->points, input_bytes(in), cudaMemcpyHostToDevice, st));
    dpts = ctx->pts.p;
  }
  GS_CK(cudaMemsetAsync(ctx->ctl.p, 0, ctl_zero_bytes(ctx->ctl_nf), st));
  ctx->ctl_clean = false;
  GS_CK(cudaMemcpyAsync(ctx->dbox.p, &b, sizeof(GsBox), cudaMemcpyHostToDevice, st));
  ctx->box = b;
  GS_TRY(dispatch_bounds_bin(ctx, dpts, in->dtype, d, n, false, 0));
  k_epoch_bump<<<1, 1, 0, st>>>(ctx->epoch_dev.as<unsigned>());
  GS_LAUNCHED("k_epoch_bump");
  unsigned* cnt32 = ctx->counters.as<unsigned>();
  const unsigned tg = (unsigned)std::min<int64_t>(sv / gs::kOccTile + 1, (int64_t)ctx->num_sms * 4);
  gs::k_occ<<<tg, 256, 0, st>>>(
      ctx->dbox.as<GsBox>(), ctx->epoch_dev.as<unsigned>(), ctx->tiles.as<unsigned long long>(),
      cnt32 + 5, cnt32, ctx->cnt.as<uint32_t>(), ctx->qs.as<unsigned long long>(),
      ctx->ckey[0].as<uint32_t>(), ctx->ccnt[0].as<uint32_t>(), ctx->S[0].as<double>(),
      ctx->idx.as<int32_t>(), ctx->root.as<int32_t>(), ctx->initkey.as<uint32_t>(),
      ctx->ifirst.as<int32_t>(), ctx->errflag.as<int>(), ctx->xsum.as<long long>());
  GS_LAUNCHED("k_occ");
  int hdr[8];
  unsigned ctr[16];
  GS_CK(cudaMemcpyAsync(hdr, ctx->errflag.p, 32, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(ctr, ctx->counters.p, 64, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaStreamSynchronize(st));
  if (hdr[0] & 2)
    return fail(ctx, GS_E_INVALID_PARAMETER, "shard points outside the given key bounds");
  const int64_t m = ctr[0];
  *m_out = m;
  if (m > cap) return fail(ctx, GS_E_INVALID_PARAMETER, "partial-cell buffers too small");
  GS_CK(cudaMemcpyAsync(keys, ctx->ckey[0].p, 4 * m, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(counts, ctx->ccnt[0].p, 4 * m, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(sums, ctx->xsum.p, 8 * d * m, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaStreamSynchronize(st));
  ctx->box = b;
  ctx->shard_box = true;
  ctx->ctl_clean = false;
  return GS_OK;
}

gs_status gs_shard_run(gs_ctx* ctx, int64_t m_all, const uint32_t* keys, const uint32_t* counts,
                       const int64_t* sums, int64_t n_shard, const gs_config* cfg,
                       gs_result* out) {
  if (!ctx || !cfg || !out || m_all < 1 || !keys || !counts || !sums)
    return GS_E_INVALID_PARAMETER;
  if (!ctx->shard_box) return fail(ctx, GS_E_INVALID_PARAMETER, "gs_shard_bin first");
  if (cfg->h != ctx->box.h) return fail(ctx, GS_E_INVALID_PARAMETER, "h differs from gs_shard_bin");
  if (n_shard != ctx->box.n) return fail(ctx, GS_E_INVALID_PARAMETER, "shard size differs");
  gs_input in{keys, n_shard, ctx->box.d, GS_F64, 1, 1, 0};  // points unused: cells given
  gs_status s = validate(&in, cfg);
  if (s != GS_OK) return s;
  ctx->err.clear();
  if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, GS_E_CUDA, "cudaSetDevice");
  ctx->shard_front = true;
  ctx->shard_m = m_all;
  ctx->shard_keys = keys;
  ctx->shard_counts = counts;
  ctx->shard_sums = sums;
  s = run_impl(ctx, &in, cfg, out);
  ctx->shard_front = false;
  ctx->shard_box = false;
  ctx->shard_keys = ctx->shard_counts = nullptr;
  ctx->shard_sums = nullptr;
  return s;
}

gs_status gs_render(gs_ctx* ctx, int64_t frame, uint8_t* out, int32_t on_device) {
  if (!ctx || !out) return GS_E_INVALID_PARAMETER;
  if (!ctx->have_run || frame < 0 || frame >= ctx->nframes)
    return fail(ctx, GS_E_INVALID_PARAMETER, "no such frame in the last run");
  if (ctx->box.d < 3) return fail(ctx, GS_E_INVALID_PARAMETER, "render needs rgb features");
  if (ctx->grouped && frame < ctx->group_f0)
    return fail(ctx, GS_E_INVALID_PARAMETER,
                "render after a pipelined run: only the last frame group is on the device");
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  const int64_t n = ctx->box.n, k = ctx->h_k[frame];
  const int64_t lf = ctx->grouped ? frame - ctx->group_f0 : frame;  // frame of the live state
  GS_TRY(grow(ctx, ctx->pkeys, 4 * (size_t)std::max<int64_t>(k, 1)));  // colour table
  uint8_t* dout = out;
  if (!on_device) {
    GS_TRY(grow(ctx, ctx->labels, 3 * (size_t)n));
    dout = ctx->labels.as<uint8_t>();
  }
  gs::k_segment_colours<<<blocks_for(k, 128), 128, 0, st>>>(
      k, ctx->box.d, ctx->S[ctx->cur].as<double>() + (size_t)ctx->h_ffirst[lf] * ctx->box.d,
      ctx->pkeys.as<uint32_t>());
  GS_LAUNCHED("k_segment_colours");
  gs::k_render<<<blocks_for(n, 256, (int64_t)ctx->num_sms * 8), 256, 0, st>>>(
      n, ctx->slot.p, lf, ctx->dbox.as<GsBox>(), ctx->lab.as<int32_t>(),
      ctx->pkeys.as<uint32_t>(), dout);
  GS_LAUNCHED("k_render");
  if (!on_device)
    GS_CK(cudaMemcpyAsync(out, dout, 3 * (size_t)n, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaStreamSynchronize(st));
  return GS_OK;
}

gs_status gs_debug_build(gs_ctx* ctx, const gs_input* in, double h, int64_t cap_m,
                         int64_t* m_out, int64_t* keys, int64_t* counts, double* centroids,
                         int64_t* slot) {
  gs_config cfg{h, 1, 0};
  GS_TRY(validate(in, &cfg));
  if (!ctx) return GS_E_INVALID_PARAMETER;
  if (in->batch != 1) return fail(ctx, GS_E_INVALID_PARAMETER, "debug build takes one frame");
  ctx->img_w = img_width(in);
  cudaSetDevice(ctx->device);
  const int d = in->d;
  const int64_t n = in->n;
  const void* dpts = in->points;
  if (!in->on_device) {
    GS_TRY(grow(ctx, ctx->pts, input_bytes(in)));
    GS_CK(cudaMemcpyAsync(ctx->pts.p, in->points, input_bytes(in), cudaMemcpyHostToDevice,
                          ctx->stream));
    dpts = ctx->pts.p;
  }
  GS_TRY(grow(ctx, ctx->errflag, 32));
  GS_TRY(grow(ctx, ctx->counters, 64));
  int64_t m0 = 0;
  for (int attempt = 0;; ++attempt) {
    GS_TRY(launch_nscale(ctx, dpts, in->dtype, d, n, 1, h));
    int hdr[8];
    unsigned ctr[16];
    GS_CK(cudaMemcpyAsync(hdr, ctx->errflag.p, 32, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CK(cudaMemcpyAsync(ctr, ctx->counters.p, 64, cudaMemcpyDeviceToHost, ctx->stream));
    GS_CK(cudaMemcpyAsync(&ctx->box, ctx->dbox.p, sizeof(GsBox), cudaMemcpyDeviceToHost,
                          ctx->stream));
    GS_CK(cudaStreamSynchronize(ctx->stream));
    if ((hdr[0] & 32) && attempt < 3) {
      GS_TRY(grow_dense_for(ctx, *(long long*)(hdr + 2), d));
      continue;
    }
    if (hdr[0] & 1) return fail(ctx, GS_E_INVALID_INPUT, "non-finite coordinate in input");
    if (hdr[0] & (32 | 64)) return fail(ctx, GS_E_KEY_RANGE, "key box too large");
    m0 = ctr[0];
    break;
  }
  *m_out = m0;
  if (m0 > cap_m) return fail(ctx, GS_E_INVALID_PARAMETER, "cap_m too small");
  std::vector<uint32_t> hk(m0), hc(m0);
  GS_CK(cudaMemcpyAsync(hk.data(), ctx->ckey[0].p, 4 * m0, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(hc.data(), ctx->ccnt[0].p, 4 * m0, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(centroids, ctx->S[0].p, sizeof(double) * m0 * d, cudaMemcpyDeviceToHost,
                        ctx->stream));
  GS_TRY(grow(ctx, ctx->dbg, sizeof(int64_t) * n));
  gs::k_slot_rank<<<blocks_for(n, 256), 256, 0, ctx->stream>>>(
      n, ctx->slot.p, ctx->dbox.as<GsBox>(), ctx->idx.as<int32_t>(), ctx->dbg.as<int64_t>());
  GS_CK(cudaGetLastError());
  GS_CK(cudaMemcpyAsync(slot, ctx->dbg.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost,
                        ctx->stream));
  gs::k_idx_clear<<<blocks_for(m0, 256), 256, 0, ctx->stream>>>(
      (int)m0, ctx->ckey[0].as<uint32_t>(), ctx->idx.as<int32_t>());
  GS_CK(cudaGetLastError());
  GS_CK(cudaStreamSynchronize(ctx->stream));
  const GsBox& b = ctx->box;
  for (int64_t i = 0; i < m0; ++i) {
    int64_t local = hk[i] % b.vol_frame;
    for (int c = 0; c < d; ++c) keys[i * d + c] = (local / b.stride[c]) % b.ext[c] + b.kmin[c];
    counts[i] = hc[i];
  }
  return GS_OK;
}

gs_status gs_debug_iterate_once(gs_ctx* ctx, int32_t d, double h, int64_t m, const int64_t* keys,
                                const int64_t* counts, const double* centroids, int64_t* m_out,
                                int64_t* keys_out, int64_t* counts_out, double* centroids_out,
                                double* swept_out, int64_t* parent_out, int32_t* changed_out,
                                int32_t* converged_out, double* maxdisp_out) {
  if (!ctx) return GS_E_INVALID_PARAMETER;
  if (!(h > 0.0) || !std::isfinite(h)) return fail(ctx, GS_E_INVALID_BANDWIDTH, "h");
  if (m < 1) return fail(ctx, GS_E_EMPTY_INPUT, "m");
  if (d < 1 || d > GS_MAX_DIM) return fail(ctx, GS_E_INVALID_PARAMETER, "d");
  cudaSetDevice(ctx->device);
  GsBox b;
  GS_TRY(make_box_from_cells(ctx, d, h, m, keys, centroids, &b));
  ctx->box = b;
  GS_TRY(ensure_dense(ctx, b.vol_total, d));
  GS_TRY(ensure_cells(ctx, m, d));
  GS_TRY(ensure_frames(ctx, 1));
  GS_TRY(grow(ctx, ctx->errflag, sizeof(int) * 4));
  GS_TRY(grow(ctx, ctx->counters, sizeof(unsigned int) * 16));
  GS_CK(cudaMemsetAsync(ctx->errflag.p, 0, sizeof(int) * 4, ctx->stream));
  ctx->ctl_clean = false;
  std::vector<uint32_t> hk(m), hc(m);
  std::vector<int32_t> hidx(m);
  for (int64_t i = 0; i < m; ++i) {
    int64_t L = 0;
    for (int c = 0; c < d; ++c) L += (keys[i * d + c] - b.kmin[c]) * b.stride[c];
    hk[i] = (uint32_t)L;
    hc[i] = (uint32_t)counts[i];
    if (i > 0 && hk[i] <= hk[i - 1])
      return fail(ctx, GS_E_INVALID_INPUT, "injected keys must be strictly lex-sorted");
  }
  ctx->cur = 0;
  GS_CK(cudaMemcpyAsync(ctx->ckey[0].p, hk.data(), 4 * m, cudaMemcpyHostToDevice, ctx->stream));
  GS_CK(cudaMemcpyAsync(ctx->ccnt[0].p, hc.data(), 4 * m, cudaMemcpyHostToDevice, ctx->stream));
  GS_CK(cudaMemcpyAsync(ctx->S[0].p, centroids, sizeof(double) * m * d, cudaMemcpyHostToDevice,
                        ctx->stream));
  GS_CK(cudaMemsetAsync(ctx->fdone.p, 0, sizeof(int32_t), ctx->stream));
  gs::k_idx_set<<<blocks_for(m, 256), 256, 0, ctx->stream>>>((int)m, ctx->ckey[0].as<uint32_t>(),
                                                             ctx->idx.as<int32_t>());
  GS_CK(cudaGetLastError());
  int64_t mnew = 0;
  GS_TRY(iterate(ctx, m, &mnew));
  int err = 0;
  GS_TRY(read_err(ctx, &err));
  if (err & 8) return fail(ctx, GS_E_INTERNAL_INVARIANT, "sweep dataflow watchdog fired");
  if (err & 4) return fail(ctx, GS_E_INTERNAL_INVARIANT, "centroid left the key box");
  std::vector<uint32_t> nk(mnew), nc(mnew);
  std::vector<int32_t> par(m);
  int32_t fch = 0, fadj = 0;
  unsigned long long fd = 0;
  GS_CK(cudaMemcpyAsync(nk.data(), ctx->ckey[1].p, 4 * mnew, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(nc.data(), ctx->ccnt[1].p, 4 * mnew, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(centroids_out, ctx->S[1].p, sizeof(double) * mnew * d,
                        cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(swept_out, ctx->S1.p, sizeof(double) * m * d, cudaMemcpyDeviceToHost,
                        ctx->stream));
  GS_CK(cudaMemcpyAsync(par.data(), ctx->parent.p, 4 * m, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(&fch, ctx->fchanged.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(&fadj, ctx->fadj.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  GS_CK(cudaMemcpyAsync(&fd, ctx->fdisp.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  gs::k_idx_clear<<<blocks_for(mnew, 256), 256, 0, ctx->stream>>>(
      (int)mnew, ctx->ckey[1].as<uint32_t>(), ctx->idx.as<int32_t>());
  GS_CK(cudaGetLastError());
  GS_CK(cudaStreamSynchronize(ctx->stream));
  *m_out = mnew;
  for (int64_t g = 0; g < mnew; ++g) {
    for (int c = 0; c < d; ++c) keys_out[g * d + c] = (nk[g] / b.stride[c]) % b.ext[c] + b.kmin[c];
    counts_out[g] = nc[g];
  }
  for (int64_t i = 0; i < m; ++i) parent_out[i] = par[i];
  *changed_out = fch;
  *converged_out = fadj ? 0 : 1;
  std::memcpy(maxdisp_out, &fd, sizeof(double));
  ctx->have_run = false;
  return GS_OK;
}


gs_status gs_debug_resident_once(gs_ctx* ctx, int32_t d, double h, int64_t m, const int64_t* keys,
                                 const int64_t* counts, const double* centroids, int64_t* m_out,
                                 int64_t* keys_out, int64_t* counts_out, double* centroids_out,
                                 int64_t* parent_out, int32_t* stop_out, double* maxdisp_out) {
  if (!ctx) return GS_E_INVALID_PARAMETER;
  if (!(h > 0.0) || !std::isfinite(h)) return fail(ctx, GS_E_INVALID_BANDWIDTH, "h");
  if (m < 1) return fail(ctx, GS_E_EMPTY_INPUT, "m");
  if (d < 1 || d > GS_MAX_DIM) return fail(ctx, GS_E_INVALID_PARAMETER, "d");
  if (m > resident_capacity(d))
    return fail(ctx, GS_E_INVALID_PARAMETER, "state larger than K8's capacity");
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  ctx->have_run = false;
  ctx->grouped = false;
  ctx->img_w = 0;
  GsBox b;
  GS_TRY(make_box_from_cells(ctx, d, h, m, keys, centroids, &b));
  ctx->box = b;
  GS_TRY(ensure_dense(ctx, b.vol_total, d));
  GS_TRY(ensure_cells(ctx, m, d));
  GS_TRY(ensure_frames(ctx, 1));
  GS_TRY(grow(ctx, ctx->hist, (sizeof(int64_t) + sizeof(double)) * 1));
  GS_TRY(grow(ctx, ctx->dbox, sizeof(GsBox)));
  GS_TRY(grow(ctx, ctx->labels, 16));
  Readback rb;
  GS_TRY(map_readback(ctx, 1, 1, &rb));
  std::vector<uint32_t> hk(m), hc(m);
  std::vector<int32_t> r0(m), first{0, (int32_t)m};
  for (int64_t i = 0; i < m; ++i) {
    int64_t L = 0;
    for (int c = 0; c < d; ++c) L += (keys[i * d + c] - b.kmin[c]) * b.stride[c];
    hk[i] = (uint32_t)L;
    hc[i] = (uint32_t)counts[i];
    r0[i] = (int32_t)i;
    if (i > 0 && hk[i] <= hk[i - 1])
      return fail(ctx, GS_E_INVALID_INPUT, "injected keys must be strictly lex-sorted");
  }
  // the state K3 leaves for K8: lex-sorted initial cells, the dense index, identity roots
  ctx->cur = 0;
  GS_CK(cudaMemsetAsync(ctx->ctl.p, 0, ctl_zero_bytes(ctx->ctl_nf), st));
  GS_CK(cudaMemcpyAsync(ctx->dbox.p, &b, sizeof(GsBox), cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->ckey[0].p, hk.data(), 4 * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->initkey.p, hk.data(), 4 * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->ccnt[0].p, hc.data(), 4 * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->S[0].p, centroids, sizeof(double) * m * d, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->root.p, r0.data(), 4 * m, cudaMemcpyHostToDevice, st));
  GS_CK(cudaMemcpyAsync(ctx->ifirst.p, first.data(), 8, cudaMemcpyHostToDevice, st));
  gs::k_idx_set<<<blocks_for(m, 256), 256, 0, st>>>((int)m, ctx->ckey[0].as<uint32_t>(),
                                                    ctx->idx.as<int32_t>());
  GS_CK(cudaGetLastError());
  ctx->ctl_clean = false;
  int ms_run = 32;
  while (ms_run < m) ms_run <<= 1;
  gs_config cfg{h, 1, GS_RECORD_HISTORY};
  ctx->ev_mask = 0;
  GS_TRY(launch_tail(ctx, &cfg, 1, 0, d, ms_run, false, true, ctx->labels.as<int32_t>(), true,
                     true, rb));
  GS_CK(cudaStreamSynchronize(st));
  if (rb.err[0] & 8) return fail(ctx, GS_E_INTERNAL_INVARIANT, "sweep schedule watchdog fired");
  if (rb.err[0] & 4) return fail(ctx, GS_E_INTERNAL_INVARIANT, "centroid left the key box");
  if (rb.err[0] & 16) return fail(ctx, GS_E_INTERNAL_INVARIANT, "state beyond K8's capacity");
  const int64_t k = rb.fk[0], f0 = rb.fout[0];
  const int fin = 1 - ctx->cur;
  std::vector<uint32_t> nk(k), nc(k);
  std::vector<int32_t> lab(b.vol_total);
  GS_CK(cudaMemcpyAsync(nk.data(), ctx->ckey[fin].as<uint32_t>() + f0, 4 * k, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(nc.data(), ctx->ccnt[fin].as<uint32_t>() + f0, 4 * k, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(centroids_out, ctx->S[fin].as<double>() + (size_t)f0 * d,
                        sizeof(double) * k * d, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaMemcpyAsync(lab.data(), ctx->lab.p, 4 * b.vol_total, cudaMemcpyDeviceToHost, st));
  GS_CK(cudaStreamSynchronize(st));
  *m_out = k;
  for (int64_t g = 0; g < k; ++g) {
    for (int c = 0; c < d; ++c) keys_out[g * d + c] = (nk[g] / b.stride[c]) % b.ext[c] + b.kmin[c];
    counts_out[g] = nc[g];
  }
  for (int64_t i = 0; i < m; ++i) parent_out[i] = lab[hk[i]];
  *stop_out = rb.fconv[0];
  *maxdisp_out = rb.hd[0];
  ctx->ctl_clean = true;  // K7 re-zeroed the control block
  return GS_OK;
}

}  // extern "C"

// ---- multi-GPU drivers (gs_dist_*)
#include "gs_dist.cuh"
