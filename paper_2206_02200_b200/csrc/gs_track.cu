// gs_track.cu — GridShift object tracking (Algorithm 2).
//
// Reference operations (/root/reference/SPEC.md, module tracker :437-498):
//   init_tracker     SPEC.md:455-463   engine.run on the window's colours, cluster selection,
//                                      reference bin B = colour cells of the selected pixels
//   track_frame      SPEC.md:464-472   inner loop: R = window pixels whose colour cell is in B,
//                                      centre = mean of R, B = cells of R, size adaptation,
//                                      window growth when R is empty
//   track_sequence   SPEC.md:473-479   frames in order, state threaded through
// Pins T1-T5 (window pixel set, colour cell, selection, inner-loop order, sequence) are stated
// in oracle/gs_oracle.cpp; every floating-point step here is the oracle's, with _rn
// intrinsics, so windows and lost flags equal the oracle's bit for bit.
//
// Design (B200): the tracker is a sequential state machine over frames (each frame's inner loop
// starts from the previous frame's window and bin) with a few thousand to tens of thousands of
// pixels per inner iteration.  The whole sequence runs in ONE persistent kernel: one CTA keeps
// the window state and both colour-cell bitmaps in shared memory, scans the window's pixels
// straight from the frames in HBM (no host round trip between iterations or frames), reduces
// count / coordinate sums / extents with warp shuffles, and writes one window per frame.
// init_tracker runs the GPU engine (8-bit front end, GS_U8) on the window crop and builds B on
// the device.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gridshift_c.h"

namespace {

constexpr int kTrackThreads = 1024;
constexpr int kMaxBitmapWords = 12288;  // shared memory: 2 x 48 KB bitmaps (K^3 <= 393,216)

__device__ __forceinline__ bool tr_range(double o, double len, int lim, int* lo, int* hi) {
  const double a = ceil(__dsub_rn(o, __dmul_rn(len, 0.5)));
  const double b = floor(__dadd_rn(o, __dmul_rn(len, 0.5)));
  const double ca = fmax(a, 0.0), cb = fmin(b, (double)(lim - 1));
  if (!(ca <= cb)) return false;
  *lo = (int)ca;
  *hi = (int)cb;
  return true;
}

// colour cell of 8-bit value v: floor((v / 255) / h), both IEEE divisions (pin T2)
__global__ void k_crop(const uint8_t* __restrict__ frame, int W, int x0, int y0, int cw, int chh,
                       uint8_t* __restrict__ crop) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= (int64_t)cw * chh) return;
  const int x = x0 + (int)(q % cw), y = y0 + (int)(q / cw);
  const uint8_t* px = frame + ((int64_t)y * W + x) * 3;
  crop[q * 3 + 0] = px[0];
  crop[q * 3 + 1] = px[1];
  crop[q * 3 + 2] = px[2];
}

__device__ __forceinline__ int tr_value_cell(int v, double h) {
  return (int)floor(__ddiv_rn(__ddiv_rn((double)v, 255.0), h));
}

// init: B = colour cells of the crop pixels whose cluster is selected
__global__ void k_init_bin(const uint8_t* __restrict__ crop, int64_t np,
                           const int32_t* __restrict__ labels, const uint8_t* __restrict__ sel,
                           double h, int K, unsigned* __restrict__ B) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= np || !sel[labels[q]]) return;
  int id = 0;
  for (int c = 0; c < 3; ++c) id = id * K + tr_value_cell(crop[q * 3 + c], h);
  atomicOr(&B[id >> 5], 1u << (id & 31));
}

struct TrackParams {
  const uint8_t* frames;  // T frames, H x W x 3
  int64_t T;
  int H, W, K, nwords, max_inner;
  double h, f, eta;
  double* state;        // [ox, oy, l, w] in / out
  unsigned* B;          // nwords in / out (the bin carried between calls)
  double* out_win;      // T x 4
  int32_t* out_lost;    // T
  int32_t* out_inner;   // T
};

__global__ void __launch_bounds__(kTrackThreads, 1) k_track(TrackParams P) {
  extern __shared__ unsigned tsm[];
  unsigned* bm0 = tsm;
  unsigned* bm1 = tsm + P.nwords;
  __shared__ int kv[256];
  __shared__ double st[4];
  __shared__ int reg[5];  // a0, a1, b0, b1, valid
  __shared__ int s_done;
  __shared__ long long wsum[32][3];
  __shared__ int wext[32][4];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int K = P.K, W = P.W;
  for (int v = tid; v < 256; v += blockDim.x) kv[v] = tr_value_cell(v, P.h);
  for (int j = tid; j < P.nwords; j += blockDim.x) bm0[j] = P.B[j];
  if (tid < 4) st[tid] = P.state[tid];
  unsigned* B = bm0;
  unsigned* NB = bm1;
  __syncthreads();
  for (int64_t t = 0; t < P.T; ++t) {
    const uint8_t* fr = P.frames + t * (int64_t)P.H * W * 3;
    bool found = false;  // meaningful in thread 0
    int inner = 0;
    for (int it = 0; it < P.max_inner; ++it) {
      ++inner;
      if (tid == 0) {
        int a0 = 0, a1 = -1, b0 = 0, b1 = -1;
        const bool ok = tr_range(st[0], __ddiv_rn(st[2], P.f), W, &a0, &a1) &&
                        tr_range(st[1], __ddiv_rn(st[3], P.f), P.H, &b0, &b1);
        reg[0] = a0;
        reg[1] = a1;
        reg[2] = b0;
        reg[3] = b1;
        reg[4] = ok ? 1 : 0;
      }
      for (int j = tid; j < P.nwords; j += blockDim.x) NB[j] = 0u;
      __syncthreads();
      long long cnt = 0, sx = 0, sy = 0;
      int mnx = INT_MAX, mxx = -1, mny = INT_MAX, mxy = -1;
      if (reg[4]) {
        const int a0 = reg[0], b0 = reg[2], rw = reg[1] - reg[0] + 1;
        const int npix = rw * (reg[3] - reg[2] + 1);
        for (int p = tid; p < npix; p += blockDim.x) {
          const int y = b0 + p / rw, x = a0 + p % rw;
          const uint8_t* px = fr + ((int64_t)y * W + x) * 3;
          const int cell = (kv[px[0]] * K + kv[px[1]]) * K + kv[px[2]];
          if (!((B[cell >> 5] >> (cell & 31)) & 1u)) continue;
          ++cnt;
          sx += x;
          sy += y;
          mnx = min(mnx, x);
          mxx = max(mxx, x);
          mny = min(mny, y);
          mxy = max(mxy, y);
          // (a solid object puts the whole window into a few cells: test before the atomic, so
          // only the first pixels of a cell pay the same-address serialisation)
          const unsigned bitm = 1u << (cell & 31);
          if (!(*(volatile unsigned*)&NB[cell >> 5] & bitm)) atomicOr(&NB[cell >> 5], bitm);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        sx += __shfl_xor_sync(0xffffffffu, sx, o);
        sy += __shfl_xor_sync(0xffffffffu, sy, o);
        mnx = min(mnx, __shfl_xor_sync(0xffffffffu, mnx, o));
        mxx = max(mxx, __shfl_xor_sync(0xffffffffu, mxx, o));
        mny = min(mny, __shfl_xor_sync(0xffffffffu, mny, o));
        mxy = max(mxy, __shfl_xor_sync(0xffffffffu, mxy, o));
      }
      if (lane == 0) {
        wsum[wid][0] = cnt;
        wsum[wid][1] = sx;
        wsum[wid][2] = sy;
        wext[wid][0] = mnx;
        wext[wid][1] = mxx;
        wext[wid][2] = mny;
        wext[wid][3] = mxy;
      }
      __syncthreads();
      if (tid == 0) {
        cnt = sx = sy = 0;
        mnx = mny = INT_MAX;
        mxx = mxy = -1;
        for (int k = 0; k < nw; ++k) {
          cnt += wsum[k][0];
          sx += wsum[k][1];
          sy += wsum[k][2];
          mnx = min(mnx, wext[k][0]);
          mxx = max(mxx, wext[k][1]);
          mny = min(mny, wext[k][2]);
          mxy = max(mxy, wext[k][3]);
        }
        int done = 0, swap = 0;
        if (cnt == 0) {  // grow (Alg. 2 lines 9-10)
          st[2] = __dmul_rn(st[2], 1.1);
          st[3] = __dmul_rn(st[3], 1.1);
        } else {
          found = true;
          swap = 1;
          const double nx = __ddiv_rn((double)sx, (double)cnt);
          const double ny = __ddiv_rn((double)sy, (double)cnt);
          st[2] = ((double)(mxx - mnx) < st[2]) ? __dmul_rn(st[2], 0.99) : __dmul_rn(st[2], 1.01);
          st[3] = ((double)(mxy - mny) < st[3]) ? __dmul_rn(st[3], 0.99) : __dmul_rn(st[3], 1.01);
          const double dx = __dsub_rn(nx, st[0]), dy = __dsub_rn(ny, st[1]);
          const double disp = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
          st[0] = nx;
          st[1] = ny;
          done = disp < P.eta;
        }
        s_done = done | (swap << 1);
      }
      __syncthreads();
      const int sd = s_done;
      if (sd & 2) {  // B <- cells of R
        unsigned* tmp = B;
        B = NB;
        NB = tmp;
      }
      if (sd & 1) break;
    }
    if (tid == 0) {
      for (int c = 0; c < 4; ++c) P.out_win[t * 4 + c] = st[c];
      P.out_lost[t] = found ? 0 : 1;
      P.out_inner[t] = inner;
    }
    __syncthreads();  // reg / st of the next frame
  }
  for (int j = tid; j < P.nwords; j += blockDim.x) P.B[j] = B[j];
  if (tid < 4) P.state[tid] = st[tid];
}

struct TDev {
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
  ~TDev() {
    if (p) cudaFree(p);
  }
};

}  // namespace

struct gs_tracker {
  int device = 0;
  cudaStream_t st = nullptr;
  gs_ctx* eng = nullptr;
  std::string err;
  bool ready = false;
  int H = 0, W = 0, K = 0, nwords = 0;
  gs_tracker_config cfg{};
  TDev crop, labels, sel, bin, state, frames, win, lost, inner;
};

namespace {

gs_status trfail(gs_tracker* t, gs_status s, const std::string& m) {
  t->err = m;
  return s;
}

#define TRCK(call)                                                              \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return trfail(t, e_ == cudaErrorMemoryAllocation ? GS_E_OOM : GS_E_CUDA,  \
                    std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

bool host_range(double o, double len, int lim, int* lo, int* hi) {
  const double a = std::ceil(o - len * 0.5), b = std::floor(o + len * 0.5);
  const double ca = std::max(a, 0.0), cb = std::min(b, (double)(lim - 1));
  if (!(ca <= cb)) return false;
  *lo = (int)ca;
  *hi = (int)cb;
  return true;
}

}  // namespace

extern "C" {

gs_status gs_tracker_create(int device, gs_tracker** out) {
  if (!out) return GS_E_INVALID_PARAMETER;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return GS_E_NO_DEVICE;
  }
  if (cudaSetDevice(device) != cudaSuccess) return GS_E_NO_DEVICE;
  gs_tracker* t = new gs_tracker();
  t->device = device;
  gs_status s = GS_OK;
  if (cudaStreamCreateWithFlags(&t->st, cudaStreamNonBlocking) != cudaSuccess) s = GS_E_CUDA;
  if (s == GS_OK) s = gs_create(device, (void*)t->st, &t->eng);
  if (s == GS_OK &&
      cudaFuncSetAttribute(k_track, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           2 * kMaxBitmapWords * 4) != cudaSuccess)
    s = GS_E_CUDA;
  if (s != GS_OK) {
    gs_tracker_destroy(t);
    return s;
  }
  *out = t;
  return GS_OK;
}

void gs_tracker_destroy(gs_tracker* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  if (t->eng) gs_destroy(t->eng);
  if (t->st) {
    cudaStreamSynchronize(t->st);
    cudaStreamDestroy(t->st);
  }
  delete t;
}

const char* gs_tracker_last_error(const gs_tracker* t) { return t ? t->err.c_str() : "null tracker"; }

gs_status gs_track_init(gs_tracker* t, const uint8_t* frame0, int32_t H, int32_t W,
                        int32_t on_device, const gs_window* win, const gs_tracker_config* cfg,
                        int64_t* k_out) {
  if (!t || !frame0 || !win || !cfg) return GS_E_INVALID_PARAMETER;
  t->err.clear();
  t->ready = false;
  if (!(cfg->h > 0.0) || !std::isfinite(cfg->h))
    return trfail(t, GS_E_INVALID_BANDWIDTH, "h must be > 0 (SPEC.md:450)");
  if (H < 1 || W < 1 || !(cfg->f >= 1.0) || !(cfg->eta > 0.0) || cfg->max_inner_iters < 1 ||
      cfg->engine_max_iter < 1 || (cfg->n_ids == 0 && cfg->top_k < 1) ||
      (cfg->n_ids > 0 && !cfg->ids) || !(win->l > 0.0) || !(win->w > 0.0))
    return trfail(t, GS_E_INVALID_PARAMETER, "tracker configuration out of range (SPEC.md:448-451)");
  const double Kd = std::floor(1.0 / cfg->h) + 1.0;
  if (!(Kd * Kd * Kd <= 32.0 * kMaxBitmapWords))
    return trfail(t, GS_E_INVALID_PARAMETER, "h too small: the colour-cell bitmap exceeds shared memory");
  int x0, x1, y0, y1;
  if (!host_range(win->ox, win->l, W, &x0, &x1) || !host_range(win->oy, win->w, H, &y0, &y1))
    return trfail(t, GS_E_INVALID_WINDOW, "window does not intersect the frame (SPEC.md:459)");
  cudaSetDevice(t->device);
  const int K = (int)Kd;
  const int nwords = (K * K * K + 31) / 32;
  const int cw = x1 - x0 + 1, chh = y1 - y0 + 1;
  const int64_t np = (int64_t)cw * chh;
  const uint8_t* dframe = frame0;
  if (!on_device) {
    TRCK(t->frames.grow((size_t)H * W * 3));
    TRCK(cudaMemcpyAsync(t->frames.p, frame0, (size_t)H * W * 3, cudaMemcpyHostToDevice, t->st));
    dframe = t->frames.as<uint8_t>();
  }
  TRCK(t->crop.grow((size_t)np * 3));
  TRCK(t->labels.grow(sizeof(int32_t) * np));
  const unsigned nb = (unsigned)((np + 255) / 256);
  k_crop<<<nb, 256, 0, t->st>>>(dframe, W, x0, y0, cw, chh, t->crop.as<uint8_t>());
  TRCK(cudaGetLastError());
  // engine.run on the window's colours (GS_U8: features (r,g,b)/255 formed on the device)
  gs_input in{t->crop.p, np, 3, GS_U8, 1, 1, 0};
  gs_config c{cfg->h, cfg->engine_max_iter, GS_DEVICE_OUTPUTS};
  int64_t k = 0;
  int32_t it = 0, cv = 0;
  gs_result r{t->labels.as<int32_t>(), &k, &it, &cv};
  gs_status s = gs_run(t->eng, &in, &c, &r);
  if (s != GS_OK) return trfail(t, s, gs_last_error(t->eng));
  // selection (pin T3): cluster sizes from the labels, top_k or explicit ids
  std::vector<int32_t> lab(np);
  TRCK(cudaMemcpyAsync(lab.data(), t->labels.p, sizeof(int32_t) * np, cudaMemcpyDeviceToHost, t->st));
  TRCK(cudaStreamSynchronize(t->st));
  std::vector<int64_t> size(k, 0);
  for (int64_t q = 0; q < np; ++q) ++size[lab[q]];
  std::vector<uint8_t> sel(k, 0);
  if (cfg->n_ids > 0) {
    for (int32_t i = 0; i < cfg->n_ids; ++i) {
      if (cfg->ids[i] < 0 || cfg->ids[i] >= k)
        return trfail(t, GS_E_SELECTION, "selected cluster id does not exist (SPEC.md:459)");
      sel[cfg->ids[i]] = 1;
    }
  } else {
    std::vector<int64_t> ord(k);
    for (int64_t q = 0; q < k; ++q) ord[q] = q;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return size[a] > size[b]; });
    for (int64_t q = 0; q < std::min<int64_t>(cfg->top_k, k); ++q) sel[ord[q]] = 1;
  }
  TRCK(t->sel.grow(k));
  TRCK(t->bin.grow(sizeof(unsigned) * nwords));
  TRCK(t->state.grow(sizeof(double) * 4));
  TRCK(cudaMemcpyAsync(t->sel.p, sel.data(), k, cudaMemcpyHostToDevice, t->st));
  TRCK(cudaMemsetAsync(t->bin.p, 0, sizeof(unsigned) * nwords, t->st));
  k_init_bin<<<nb, 256, 0, t->st>>>(t->crop.as<uint8_t>(), np, t->labels.as<int32_t>(),
                                    t->sel.as<uint8_t>(), cfg->h, K, t->bin.as<unsigned>());
  TRCK(cudaGetLastError());
  const double st0[4] = {win->ox, win->oy, win->l, win->w};
  TRCK(cudaMemcpyAsync(t->state.p, st0, sizeof(st0), cudaMemcpyHostToDevice, t->st));
  TRCK(cudaStreamSynchronize(t->st));
  t->H = H;
  t->W = W;
  t->K = K;
  t->nwords = nwords;
  t->cfg = *cfg;
  t->cfg.ids = nullptr;
  t->ready = true;
  if (k_out) *k_out = k;
  return GS_OK;
}

gs_status gs_track_sequence(gs_tracker* t, const uint8_t* frames, int64_t T, int32_t on_device,
                            gs_window* out, int32_t* lost, int32_t* inner) {
  if (!t || !frames || !out || T < 1) return GS_E_INVALID_PARAMETER;
  t->err.clear();
  if (!t->ready) return trfail(t, GS_E_INVALID_PARAMETER, "gs_track_init first");
  cudaSetDevice(t->device);
  const size_t fbytes = (size_t)t->H * t->W * 3;
  const uint8_t* dfr = frames;
  if (!on_device) {
    TRCK(t->frames.grow(fbytes * T));
    TRCK(cudaMemcpyAsync(t->frames.p, frames, fbytes * T, cudaMemcpyHostToDevice, t->st));
    dfr = t->frames.as<uint8_t>();
  }
  TRCK(t->win.grow(sizeof(double) * 4 * T));
  TRCK(t->lost.grow(sizeof(int32_t) * T));
  TRCK(t->inner.grow(sizeof(int32_t) * T));
  TrackParams P;
  P.frames = dfr;
  P.T = T;
  P.H = t->H;
  P.W = t->W;
  P.K = t->K;
  P.nwords = t->nwords;
  P.max_inner = t->cfg.max_inner_iters;
  P.h = t->cfg.h;
  P.f = t->cfg.f;
  P.eta = t->cfg.eta;
  P.state = t->state.as<double>();
  P.B = t->bin.as<unsigned>();
  P.out_win = t->win.as<double>();
  P.out_lost = t->lost.as<int32_t>();
  P.out_inner = t->inner.as<int32_t>();
  k_track<<<1, kTrackThreads, 2 * sizeof(unsigned) * t->nwords, t->st>>>(P);
  TRCK(cudaGetLastError());
  static_assert(sizeof(gs_window) == 4 * sizeof(double), "gs_window layout");
  TRCK(cudaMemcpyAsync(out, t->win.p, sizeof(double) * 4 * T, cudaMemcpyDeviceToHost, t->st));
  if (lost)
    TRCK(cudaMemcpyAsync(lost, t->lost.p, sizeof(int32_t) * T, cudaMemcpyDeviceToHost, t->st));
  if (inner)
    TRCK(cudaMemcpyAsync(inner, t->inner.p, sizeof(int32_t) * T, cudaMemcpyDeviceToHost, t->st));
  TRCK(cudaStreamSynchronize(t->st));
  return GS_OK;
}

}  // extern "C"
