// gs_tune.cu — bandwidth sweep: tune_bandwidth + silhouette_subsampled.
//
// Reference operations (/root/reference/SPEC.md, module metrics):
//   silhouette
//   tune_bandwidth          SPEC.md:319-327 (grid default :347, normalisation :348)
//   silhouette_subsampled
// The pins the SPEC leaves open (S1 subsample, S2 silhouette summation order, S3 undefined
// entries and ties) are stated in oracle/gs_oracle.cpp and DESIGN.md §"Bandwidth sweep"; this
// file follows them to the bit.
//
// Design (B200): the sweep entries are independent engine runs (SPEC.md "Bandwidth sweep
// entries may evaluate concurrently with isolated clusterer state"), and one run of an
// image-sized input occupies a handful of SMs for most of its time (the CTA-resident
// iteration engine runs one CTA per frame).  So a gs_tuner owns several engine contexts, each
// on its own stream and host thread, and runs the h values concurrently on one GPU: the
// points are uploaded once and shared read-only; each entry's silhouette is computed on the
// GPU right after its run, on the same stream.  Silhouette kernel: one thread per sample
// point walks the label-sorted sample in the pinned order (S2), the sample tile broadcast
// from shared memory; fp64 distances with explicit _rn intrinsics (no FMA), so the per-point
// values equal the oracle's bit for bit and the score (summed on the host in sample order)
// does too.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "gridshift_c.h"

namespace {

constexpr int kSilThreads = 64;

uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// pin S1: every point when n <= cap, else a sparse partial Fisher-Yates, sorted ascending
std::vector<int64_t> sample_indices(int64_t n, int64_t cap, uint64_t seed) {
  std::vector<int64_t> out;
  if (n <= cap) {
    out.resize(n);
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    return out;
  }
  out.resize(cap);
  std::unordered_map<int64_t, int64_t> sw;
  auto at = [&](int64_t i) {
    auto it = sw.find(i);
    return it == sw.end() ? i : it->second;
  };
  uint64_t st = seed;
  for (int64_t i = 0; i < cap; ++i) {
    const int64_t j = i + (int64_t)(splitmix64(st) % (uint64_t)(n - i));
    const int64_t vi = at(i), vj = at(j);
    sw[i] = vj;
    sw[j] = vi;
    out[i] = vj;
  }
  std::sort(out.begin(), out.end());
  return out;
}

template <typename T>
__global__ void k_gather_points(const T* __restrict__ pts, const int64_t* __restrict__ idx,
                                int64_t s, int d, double* __restrict__ xs) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= s) return;
  for (int c = 0; c < d; ++c) xs[t * d + c] = (double)pts[idx[t] * d + c];
}

__global__ void k_gather_labels(const int32_t* __restrict__ labels,
                                const int64_t* __restrict__ idx, int64_t s,
                                int32_t* __restrict__ ls) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < s) ls[t] = labels[idx[t]];
}

// Xo = the sample in label-sorted order (ord), for contiguous broadcast reads
__global__ void k_permute(const double* __restrict__ xs, const int32_t* __restrict__ ord,
                          int64_t s, int d, double* __restrict__ xo) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= s) return;
  for (int c = 0; c < d; ++c) xo[t * d + c] = xs[(int64_t)ord[t] * d + c];
}

__device__ __forceinline__ double gs_dist(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int c = 0; c < d; ++c) {
    const double t = __dsub_rn(a[c], b[c]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return __dsqrt_rn(acc);
}

// silhouette (pin S2), parallel over (sample point, cluster) pairs: CTA (x, c) gives its
// kSilThreads sorted positions the mean distance to the members of cluster c, summed in the
// members' sorted order (the pinned order: each pair's sum is the same chain as the serial
// walk's), with u itself skipped in its own cluster.  The own cluster's mean is a(u); the other
// clusters' means meet in an atomic min on the bits of b(u) (non-negative doubles order as
// their bit patterns), so b(u) is the exact minimum in any order.  Members are staged in shared
// memory and read as a broadcast.  seg[0..kc] = cluster starts in sorted order; cid[u] = u's
// cluster.  (One thread per point walking every cluster left 97 % of the warp slots idle.)
template <int D>
__global__ void __launch_bounds__(kSilThreads) k_silhouette(
    const double* __restrict__ xo, int64_t s, int d_rt, const int32_t* __restrict__ seg, int kc,
    const int32_t* __restrict__ cid, double* __restrict__ amean,
    unsigned long long* __restrict__ bmin, int c0) {
  constexpr int DD = D > 0 ? D : 12;
  constexpr int kSilTile = 4096 / DD;  // members staged per round (32 KB)
  const int d = D > 0 ? D : d_rt;
  __shared__ double tile[kSilTile * DD];
  const int c = c0 + (int)blockIdx.y;
  const int64_t cs = seg[c], ce = seg[c + 1], size = ce - cs;
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = u < s;
  double xi[DD];
  for (int k = 0; k < d; ++k) xi[k] = live ? xo[u * d + k] : 0.0;
  const int own = live ? cid[u] : -1;
  double sum = 0.0;
  for (int64_t t0 = cs; t0 < ce; t0 += kSilTile) {
    const int64_t nt = min((int64_t)kSilTile, ce - t0);
    __syncthreads();
    for (int64_t e = threadIdx.x; e < nt * d; e += blockDim.x) tile[e] = xo[t0 * d + e];
    __syncthreads();
    for (int64_t tt = 0; tt < nt; ++tt)
      if (t0 + tt != u) sum = __dadd_rn(sum, gs_dist(xi, tile + tt * d, d));
  }
  if (!live) return;
  if (c == own) {
    amean[u] = size == 1 ? -1.0 : __ddiv_rn(sum, (double)(size - 1));  // -1: a singleton
  } else {
    atomicMin(&bmin[u], (unsigned long long)__double_as_longlong(__ddiv_rn(sum, (double)size)));
  }
}

__global__ void k_sil_init(int64_t s, unsigned long long* __restrict__ bmin) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < s) bmin[u] = 0x7ff0000000000000ull;  // +inf
}

__global__ void k_sil_combine(int64_t s, const int32_t* __restrict__ ord,
                              const double* __restrict__ amean,
                              const unsigned long long* __restrict__ bmin,
                              double* __restrict__ sil) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= s) return;
  const double a0 = amean[u], b = __longlong_as_double((long long)bmin[u]);
  const bool single = a0 < 0.0;
  const double a = single ? 0.0 : a0;
  const double mx = a > b ? a : b;
  sil[ord[u]] = (single || mx == 0.0) ? 0.0 : __ddiv_rn(__dsub_rn(b, a), mx);
}

struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t grow(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  template <typename T>
  T* as() const { return (T*)p; }
  ~DevMem() {
    if (p) cudaFree(p);
  }
};

// one worker: an engine context on its own stream plus the per-entry silhouette buffers
struct Worker {
  gs_ctx* eng = nullptr;
  cudaStream_t st = nullptr;
  DevMem labels, ls, ord, seg, cid, xo, sil, amean, bmin;
  std::vector<int32_t> h_ls, h_ord, h_seg, h_cid;
  std::vector<double> h_sil;
};

}  // namespace

struct gs_tuner {
  int device = 0;
  int nwork = 1;
  std::vector<Worker> work;
  DevMem pts, idx, xs;
  std::string err;
  std::mutex mu;
};

namespace {

gs_status tfail(gs_tuner* t, gs_status s, const std::string& m) {
  std::lock_guard<std::mutex> g(t->mu);
  if (t->err.empty()) t->err = m;
  return s;
}

#define TCK(call)                                                               \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return tfail(t, e_ == cudaErrorMemoryAllocation ? GS_E_OOM : GS_E_CUDA,   \
                   std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

size_t dtype_size(int dt) { return dt == GS_F64 ? 8 : 4; }

// Stage the sample: device points (uploaded once), sample indices, gathered fp64 sample.
gs_status stage(gs_tuner* t, const gs_input* in, int64_t cap, uint64_t seed, int64_t* s_out,
                const void** dpts_out) {
  const int64_t n = in->n;
  const int d = in->d;
  const size_t bytes = (size_t)n * d * dtype_size(in->dtype);
  const void* dpts = in->points;
  cudaStream_t st = t->work[0].st;
  if (!in->on_device) {
    TCK(t->pts.grow(bytes));
    TCK(cudaMemcpyAsync(t->pts.p, in->points, bytes, cudaMemcpyHostToDevice, st));
    dpts = t->pts.p;
  }
  const std::vector<int64_t> idx = sample_indices(n, cap, seed);
  const int64_t s = (int64_t)idx.size();
  TCK(t->idx.grow(sizeof(int64_t) * s));
  TCK(t->xs.grow(sizeof(double) * s * d));
  TCK(cudaMemcpyAsync(t->idx.p, idx.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, st));
  const unsigned nb = (unsigned)((s + 255) / 256);
  if (in->dtype == GS_F64)
    k_gather_points<double><<<nb, 256, 0, st>>>((const double*)dpts, t->idx.as<int64_t>(), s, d,
                                               t->xs.as<double>());
  else
    k_gather_points<float><<<nb, 256, 0, st>>>((const float*)dpts, t->idx.as<int64_t>(), s, d,
                                              t->xs.as<double>());
  TCK(cudaGetLastError());
  TCK(cudaStreamSynchronize(st));  // every worker stream reads pts / xs from here on
  *s_out = s;
  *dpts_out = dpts;
  return GS_OK;
}

template <int D>
void launch_sil(const Worker& w, int64_t s, int d, int kc) {
  for (int c0 = 0; c0 < kc; c0 += 65535) {  // (grid.y limit)
    const dim3 grid((unsigned)((s + kSilThreads - 1) / kSilThreads), (unsigned)min(65535, kc - c0));
    k_silhouette<D><<<grid, kSilThreads, 0, w.st>>>(w.xo.as<double>(), s, d, w.seg.as<int32_t>(),
                                                   kc, w.cid.as<int32_t>(), w.amean.as<double>(),
                                                   w.bmin.as<unsigned long long>(), c0);
  }
}

// silhouette (pin S2) of the sample under the device labels `dlabels` (n entries).
gs_status silhouette_dev(gs_tuner* t, Worker& w, const int32_t* dlabels, int64_t s, int d,
                         double* score, int32_t* valid) {
  TCK(w.ls.grow(sizeof(int32_t) * s));
  const unsigned nb = (unsigned)((s + 255) / 256);
  k_gather_labels<<<nb, 256, 0, w.st>>>(dlabels, t->idx.as<int64_t>(), s, w.ls.as<int32_t>());
  TCK(cudaGetLastError());
  w.h_ls.resize(s);
  TCK(cudaMemcpyAsync(w.h_ls.data(), w.ls.p, sizeof(int32_t) * s, cudaMemcpyDeviceToHost, w.st));
  TCK(cudaStreamSynchronize(w.st));
  // label-sorted order (stable by sample position) and cluster segments
  w.h_ord.resize(s);
  for (int64_t i = 0; i < s; ++i) w.h_ord[i] = (int32_t)i;
  std::stable_sort(w.h_ord.begin(), w.h_ord.end(),
                   [&](int32_t a, int32_t b) { return w.h_ls[a] < w.h_ls[b]; });
  w.h_seg.clear();
  w.h_cid.resize(s);
  for (int64_t u = 0; u < s; ++u) {
    if (u == 0 || w.h_ls[w.h_ord[u]] != w.h_ls[w.h_ord[u - 1]]) w.h_seg.push_back((int32_t)u);
    w.h_cid[u] = (int32_t)w.h_seg.size() - 1;
  }
  const int kc = (int)w.h_seg.size();
  w.h_seg.push_back((int32_t)s);
  *score = 0.0;
  *valid = kc >= 2 ? 1 : 0;
  if (kc < 2) return GS_OK;  // S3: undefined
  TCK(w.ord.grow(sizeof(int32_t) * s));
  TCK(w.cid.grow(sizeof(int32_t) * s));
  TCK(w.seg.grow(sizeof(int32_t) * (kc + 1)));
  TCK(w.xo.grow(sizeof(double) * s * d));
  TCK(w.sil.grow(sizeof(double) * s));
  TCK(w.amean.grow(sizeof(double) * s));
  TCK(w.bmin.grow(sizeof(unsigned long long) * s));
  TCK(cudaMemcpyAsync(w.ord.p, w.h_ord.data(), sizeof(int32_t) * s, cudaMemcpyHostToDevice, w.st));
  TCK(cudaMemcpyAsync(w.cid.p, w.h_cid.data(), sizeof(int32_t) * s, cudaMemcpyHostToDevice, w.st));
  TCK(cudaMemcpyAsync(w.seg.p, w.h_seg.data(), sizeof(int32_t) * (kc + 1), cudaMemcpyHostToDevice,
                      w.st));
  k_permute<<<nb, 256, 0, w.st>>>(t->xs.as<double>(), w.ord.as<int32_t>(), s, d,
                                  w.xo.as<double>());
  k_sil_init<<<nb, 256, 0, w.st>>>(s, w.bmin.as<unsigned long long>());
  switch (d) {
    case 1: launch_sil<1>(w, s, d, kc); break;
    case 2: launch_sil<2>(w, s, d, kc); break;
    case 3: launch_sil<3>(w, s, d, kc); break;
    case 4: launch_sil<4>(w, s, d, kc); break;
    case 5: launch_sil<5>(w, s, d, kc); break;
    default: launch_sil<0>(w, s, d, kc); break;
  }
  k_sil_combine<<<nb, 256, 0, w.st>>>(s, w.ord.as<int32_t>(), w.amean.as<double>(),
                                      w.bmin.as<unsigned long long>(), w.sil.as<double>());
  TCK(cudaGetLastError());
  w.h_sil.resize(s);
  TCK(cudaMemcpyAsync(w.h_sil.data(), w.sil.p, sizeof(double) * s, cudaMemcpyDeviceToHost, w.st));
  TCK(cudaStreamSynchronize(w.st));
  double total = 0.0;
  for (int64_t i = 0; i < s; ++i) total = total + w.h_sil[i];
  *score = total / (double)s;
  return GS_OK;
}

gs_status check_input(gs_tuner* t, const gs_input* in) {
  if (!in) return GS_E_INVALID_PARAMETER;
  gs_config c{1.0, 1, 0};
  gs_status s = gs_validate(in, &c);
  if (s != GS_OK) return tfail(t, s, gs_status_string(s));
  if (in->batch != 1) return tfail(t, GS_E_INVALID_PARAMETER, "a sweep clusters one dataset");
  if (in->dtype != GS_F32 && in->dtype != GS_F64)
    return tfail(t, GS_E_INVALID_PARAMETER, "the sweep takes fp32/fp64 features");
  return GS_OK;
}

}  // namespace

extern "C" {

gs_status gs_tuner_create(int device, int32_t max_concurrent, gs_tuner** out) {
  if (!out || max_concurrent < 1) return GS_E_INVALID_PARAMETER;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return GS_E_NO_DEVICE;
  }
  if (cudaSetDevice(device) != cudaSuccess) return GS_E_NO_DEVICE;
  gs_tuner* t = new gs_tuner();
  t->device = device;
  t->nwork = max_concurrent;
  t->work.resize(max_concurrent);
  for (Worker& w : t->work) {
    gs_status s = GS_OK;
    if (cudaStreamCreateWithFlags(&w.st, cudaStreamNonBlocking) != cudaSuccess) s = GS_E_CUDA;
    if (s == GS_OK) s = gs_create(device, (void*)w.st, &w.eng);
    if (s != GS_OK) {
      gs_tuner_destroy(t);
      return s;
    }
  }
  *out = t;
  return GS_OK;
}

void gs_tuner_destroy(gs_tuner* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  for (Worker& w : t->work) {
    if (w.eng) gs_destroy(w.eng);
    if (w.st) {
      cudaStreamSynchronize(w.st);
      cudaStreamDestroy(w.st);
    }
  }
  delete t;
}

const char* gs_tuner_last_error(const gs_tuner* t) { return t ? t->err.c_str() : "null tuner"; }

gs_status gs_silhouette_subsampled(gs_tuner* t, const gs_input* X, const int32_t* labels,
                                   int32_t labels_on_device, int64_t cap, uint64_t seed,
                                   double* score) {
  if (!t || !labels || !score) return GS_E_INVALID_PARAMETER;
  t->err.clear();
  gs_status s0 = check_input(t, X);
  if (s0 != GS_OK) return s0;
  if (cap < 2) return tfail(t, GS_E_INVALID_PARAMETER, "cap must be >= 2 (SPEC.md:331)");
  cudaSetDevice(t->device);
  int64_t s;
  const void* dpts;
  gs_status st = stage(t, X, cap, seed, &s, &dpts);
  if (st != GS_OK) return st;
  Worker& w = t->work[0];
  const int32_t* dl = labels;
  if (!labels_on_device) {
    TCK(w.labels.grow(sizeof(int32_t) * X->n));
    TCK(cudaMemcpyAsync(w.labels.p, labels, sizeof(int32_t) * X->n, cudaMemcpyHostToDevice, w.st));
    dl = w.labels.as<int32_t>();
  }
  int32_t valid;
  st = silhouette_dev(t, w, dl, s, X->d, score, &valid);
  if (st != GS_OK) return st;
  if (!valid) return tfail(t, GS_E_UNDEFINED_SCORE, "fewer than 2 clusters in the sample");
  return GS_OK;
}

gs_status gs_tune_bandwidth(gs_tuner* t, const gs_input* X, const double* h_grid, int32_t nh,
                            int32_t max_iter, int64_t cap, uint64_t seed, gs_sweep_entry* out,
                            double* best_h) {
  if (!t || !h_grid || !out || !best_h) return GS_E_INVALID_PARAMETER;
  t->err.clear();
  gs_status s0 = check_input(t, X);
  if (s0 != GS_OK) return s0;
  if (nh < 1) return tfail(t, GS_E_INVALID_PARAMETER, "empty bandwidth grid (SPEC.md:322)");
  if (cap < 2) return tfail(t, GS_E_INVALID_PARAMETER, "cap must be >= 2 (SPEC.md:331)");
  if (max_iter < 1) return tfail(t, GS_E_INVALID_PARAMETER, "max_iter must be >= 1");
  for (int32_t i = 0; i < nh; ++i)
    if (!(h_grid[i] > 0.0 && h_grid[i] <= 1.0))
      return tfail(t, GS_E_INVALID_BANDWIDTH, "grid values must lie in (0, 1] (SPEC.md:322)");
  cudaSetDevice(t->device);
  int64_t s;
  const void* dpts;
  gs_status st = stage(t, X, cap, seed, &s, &dpts);
  if (st != GS_OK) return st;
  const int64_t n = X->n;
  const int d = X->d;
  std::vector<gs_status> res(nh, GS_OK);
  std::atomic<int32_t> next{0};
  auto worker = [&](int wi) {
    cudaSetDevice(t->device);
    Worker& w = t->work[wi];
    if (w.labels.grow(sizeof(int32_t) * n) != cudaSuccess) {
      for (int32_t i = next.fetch_add(1); i < nh; i = next.fetch_add(1)) res[i] = GS_E_OOM;
      return;
    }
    for (int32_t i = next.fetch_add(1); i < nh; i = next.fetch_add(1)) {
      gs_sweep_entry& e = out[i];
      e.h = h_grid[i];
      e.score = 0.0;
      e.valid = 0;
      gs_input in{dpts, n, d, X->dtype, 1, 1, 0};
      gs_config cfg{h_grid[i], max_iter, GS_DEVICE_OUTPUTS};
      int64_t k = 0;
      int32_t it = 0, cv = 0;
      gs_result r{w.labels.as<int32_t>(), &k, &it, &cv};
      gs_status rs = gs_run(w.eng, &in, &cfg, &r);
      if (rs != GS_OK) {
        res[i] = tfail(t, rs, gs_last_error(w.eng));
        continue;
      }
      e.k = k;
      e.iterations = it;
      e.converged = cv;
      res[i] = silhouette_dev(t, w, w.labels.as<int32_t>(), s, d, &e.score, &e.valid);
    }
  };
  const int nw = std::min<int>(t->nwork, nh);
  std::vector<std::thread> pool;
  for (int wi = 1; wi < nw; ++wi) pool.emplace_back(worker, wi);
  worker(0);
  for (auto& th : pool) th.join();
  for (int32_t i = 0; i < nh; ++i)
    if (res[i] != GS_OK) return res[i];  // first failing entry in grid order
  int best = -1;  // S3: max score, ties -> smallest h
  for (int32_t i = 0; i < nh; ++i)
    if (out[i].valid && (best < 0 || out[i].score > out[best].score ||
                         (out[i].score == out[best].score && out[i].h < out[best].h)))
      best = i;
  if (best < 0) return tfail(t, GS_E_TUNING_FAILED, "no bandwidth gave >= 2 clusters (SPEC.md:324)");
  *best_h = out[best].h;
  return GS_OK;
}

}  // extern "C"
