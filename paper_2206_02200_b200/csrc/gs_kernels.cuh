// gs_kernels.cuh — sm_100a kernels of the GridShift hot path (n-scale and global path).
//
//   K1 k_bounds_box     bounds, non-finite check, device key box
//   K2 k_bin_priv       grid_index + build_active_grid fixed-point sums
//   K3 k_occ            occupied cells -> lex-ordered cell list, frames
//      k_scatter_partials  multi-GPU: merge every rank's partial cells
//   K5 k_rehome, k_heads, k_seg, k_fold, k_idx_*, k_adjacent, k_compose
//                       global path: rehome + merge_into (Eq. 3-4) + has_converged
//                       (SPEC.md:67-75, :120(d-f), :126-134); the sweep is in gs_global.cuh
//   K7 k_label          label propagation through the label table
// K8 (the CTA-resident iteration engine) is gs_resident.cuh.
#pragma once

#include "gs_common.cuh"

namespace gs {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- K1: bounds + box
// Per-block min/max of every coordinate (non-finite values set err bit 1); the last block to
// finish reduces the partials and writes the dense-grid geometry, so no host round trip and
// no second launch sit between the bounds pass and binning.  err bit 32: key box larger than
// the allocated grid (*need = cells required); bit 64: keys beyond the int64 key range.
// *epoch is bumped once per run (it tags the compaction's look-back flags).
template <int D, typename T>
__global__ void __launch_bounds__(256) k_bounds_box(const T* __restrict__ pts, int64_t ntot,
                                                    double* __restrict__ bpart, double h, int F,
                                                    int64_t n, int64_t nframes,
                                                    int64_t cap_cells, GsBox* __restrict__ out,
                                                    int* err, long long* need,
                                                    unsigned* ticket, unsigned* epoch,
                                                    int img_w = 0, T* __restrict__ copy = nullptr) {
  // copy != null: `pts` is pinned host memory read over the bus (zero copy) and every point is
  // stored to `copy` (device) for K2 -- the host-to-device copy and the bounds pass are one
  constexpr int RC = gs_raw_cols<T, D>();
  const GsImg im = gs_img(img_w, n);
  double mn[D], mx[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    mn[c] = INFINITY;
    mx[c] = -INFINITY;
  }
  bool bad = false;
  auto point = [&](const T* raw, int64_t pl) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      double x = gs_feature<T, D>(raw, c, pl, im);
      bad |= !isfinite(x);
      mn[c] = fmin(mn[c], x);
      mx[c] = fmax(mx[c], x);
    }
  };
  // 16-byte vector loads: a chunk of RC words is PPC whole points (4 fp32 / 2 fp64 points,
  // 16 pixels); two chunks per thread are in flight before either is reduced
  constexpr int PPC = 16 / sizeof(T);
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((uintptr_t)pts & 15) == 0 && ((uintptr_t)copy & 15) == 0;
  const int64_t nch = vec ? ntot / PPC : 0;
  const uint4* src = reinterpret_cast<const uint4*>(pts);
  uint4* dst = reinterpret_cast<uint4*>(copy);
  for (int64_t ch = gtid; ch < nch; ch += 2 * gstride) {
    const int64_t ch1 = ch + gstride;
    const bool two = ch1 < nch;
    uint4 w0[RC], w1[RC];
#pragma unroll
    for (int r = 0; r < RC; ++r) w0[r] = src[ch * RC + r];
    if (two) {
#pragma unroll
      for (int r = 0; r < RC; ++r) w1[r] = src[ch1 * RC + r];
    }
    if (copy) {
#pragma unroll
      for (int r = 0; r < RC; ++r) dst[ch * RC + r] = w0[r];
      if (two) {
#pragma unroll
        for (int r = 0; r < RC; ++r) dst[ch1 * RC + r] = w1[r];
      }
    }
    int64_t pl = (sizeof(T) == 1 && D > 3) ? (ch * PPC) % n : 0;  // rgbxy needs the pixel index
    const T* e0 = reinterpret_cast<const T*>(w0);
#pragma unroll
    for (int j = 0; j < PPC; ++j) {
      point(e0 + j * RC, pl);
      if (sizeof(T) == 1 && D > 3 && ++pl == n) pl = 0;
    }
    if (two) {
      pl = (sizeof(T) == 1 && D > 3) ? (ch1 * PPC) % n : 0;
      const T* e1 = reinterpret_cast<const T*>(w1);
#pragma unroll
      for (int j = 0; j < PPC; ++j) {
        point(e1 + j * RC, pl);
        if (sizeof(T) == 1 && D > 3 && ++pl == n) pl = 0;
      }
    }
  }
  // points after the last whole chunk (all of them when the pointers are not 16-byte aligned)
  for (int64_t p = nch * PPC + gtid; p < ntot; p += gstride) {
    T raw[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) raw[c] = pts[p * RC + c];
    if (copy) {
#pragma unroll
      for (int c = 0; c < RC; ++c) copy[p * RC + c] = raw[c];
    }
    point(raw, (sizeof(T) == 1 && D > 3) ? p % n : 0);
  }
  if (bad) atomicOr(err, 1);
  __shared__ double smn[8][D], smx[8][D];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double a = mn[c], b = mx[c];
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(kFull, a, o));
      b = fmax(b, __shfl_xor_sync(kFull, b, o));
    }
    if (lane == 0) {
      smn[w][c] = a;
      smx[w][c] = b;
    }
  }
  __syncthreads();
  const int nblk = gridDim.x;
  if (threadIdx.x < D) {
    int c = threadIdx.x;
    double a = INFINITY, b = -INFINITY;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a = fmin(a, smn[i][c]);
      b = fmax(b, smx[i][c]);
    }
    bpart[blockIdx.x * D + c] = a;
    bpart[(nblk + blockIdx.x) * D + c] = b;
  }
  __threadfence();  // partials and error bits before the ticket
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (unsigned)nblk - 1u;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the last block: 32 lanes per dimension over the partials (L2 reads), shuffle reduction
  __shared__ double bmn[D], bmx[D];
  for (int c = w; c < D; c += blockDim.x >> 5) {
    double a = INFINITY, z = -INFINITY;
#pragma unroll 4
    for (int k = lane; k < nblk; k += 32) {
      a = fmin(a, __ldcg(&bpart[k * D + c]));
      z = fmax(z, __ldcg(&bpart[(nblk + k) * D + c]));
    }
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(kFull, a, o));
      z = fmax(z, __shfl_xor_sync(kFull, z, o));
    }
    if (lane == 0) {
      bmn[c] = a;
      bmx[c] = z;
    }
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  GsBox b;
  b.d = D;
  b.F = F;
  b.h = h;
  b.inv_h = __drcp_rn(h);
  b.scale = ldexp(1.0, F);
  b.inv_scale = ldexp(1.0, -F);
  b.n = n;
  b.nframes = nframes;
  double vol = 1.0;
  bool badk = (atomicOr(err, 0) & 1) != 0;
  for (int k = 0; k < GS_DMAX; ++k) b.kmin[k] = 0, b.ext[k] = 1, b.stride[k] = 0;
  for (int k = 0; k < D && !badk; ++k) {
    const double lo = floor(__ddiv_rn(bmn[k], h)), hi = floor(__ddiv_rn(bmx[k], h));
    if (!(fabs(lo) < 4e15) || !(fabs(hi) < 4e15)) {
      badk = true;
      break;
    }
    b.kmin[k] = (int64_t)lo - GS_APRON;
    b.ext[k] = (int64_t)hi - (int64_t)lo + 1 + 2 * GS_APRON;
    vol *= (double)b.ext[k];
  }
  int64_t s = 1;
  for (int k = D - 1; k >= 0; --k) {
    b.stride[k] = s;
    s *= b.ext[k];
  }
  b.vol_frame = s;
  b.vol_total = s * nframes;
  if (!badk && vol * (double)nframes > (double)cap_cells) {
    atomicOr(err, 32);
    *need = (vol * (double)nframes < 9e18) ? (long long)(vol * (double)nframes) : (1ll << 62);
  }
  if (badk && !(atomicOr(err, 0) & 1)) atomicOr(err, 64);  // keys beyond the int64 range
  *out = b;
  *epoch += 1u;
}

// ---------------------------------------------------------------- K2: binning
// Shared-memory privatisation: hot cells take tens of thousands of points (cfg2: 16K in one
// cell, cfg5: 415K), so per-point global atomics would serialise at one L2 slice.  Each CTA bins
// a contiguous range of points into a shared-memory table of cell accumulators (count + D int64
// fixed-point sums) and flushes it to the dense grid with global atomics.  int64 sums are
// associative, so the result is bit-identical to the oracle's build mode 1 for any schedule.
//
// Two table kinds, chosen per launch from the key box (uniformly by every CTA):
//  * dense: the frame's data box (the key box without its apron) fits the table, possibly
//    several times (replicas chosen by lane, so the hot cells of a warp spread over replica
//    entries; summed by the flush).  The CTA's range is cut at frame boundaries and the table is
//    flushed per frame.  No hashing, no probing, no key words: image frames (cfg2-4);
//  * hash: open addressing over (global cell index), bounded probes, global atomics on a miss
//    (clouds whose box is far larger than a CTA's table: cfg5).
// 64-bit shared adds are two native 32-bit atomics with the carry of the low word (sm_100 has no
// 64-bit shared add; atomicAdd(u64) compiles to a CAS loop).  Low and high words live in
// separate arrays (SoA), so a warp's entries spread over the banks.
//
// Predicted box (`predicted` != 0): the key box is the one the previous run of this shape used
// (no bounds pass); a point outside it sets err bit 128 (the host clears the grid and reruns
// with the bounds pass) and a non-finite coordinate sets bit 1.
constexpr int kBinThreads = 1024;
constexpr int kBinProbes = 4;  // hash probe budget before the point takes the global atomics
constexpr int kAggRuns = 4;    // warp aggregation when the warp's keys form <= this many runs
constexpr int kBinSmemBytes = 224 * 1024;

__device__ __forceinline__ void smem_add64(unsigned* lo, unsigned* hi, unsigned long long v) {
  const unsigned l = (unsigned)v;
  const unsigned old = atomicAdd(lo, l);
  atomicAdd(hi, (unsigned)(v >> 32) + ((old + l < old) ? 1u : 0u));
}

// grid_index of one coordinate (build mode 1), lean fp64 form of gs_grid_coord: fl =
// floor(RN(x*RN(1/h))) is final when |q| < 2^20 and q is more than 2^-30 from an integer
// (|q - x/h| <= 2^-32 there, so fl == floor(RN(x/h))), or when x == 0; otherwise the caller
// takes the IEEE quotient.  Returns whether fl needs that.
__device__ __forceinline__ bool gs_bin_floor(double x, double inv_h, double& fl) {
  const double qd = __dmul_rn(x, inv_h);
  fl = floor(qd);
  const double t = __dsub_rn(__dsub_rn(qd, fl), 0.5);
  return !(fabs(t) < 0.5 - 0x1p-30 && fabs(qd) < 0x1p20) && x != 0.0;
}

// fp32 inputs: the same floor from fp32 arithmetic.  t = RN32(x * RN32(1/h)) is within
// |t| 2^-22.9 of x/h, so when t's fractional part is farther than |t| 2^-20 + 2^-23 from 0 and
// from 1 (and |t| < 2^22), floor(t) == floor(x/h) == floor(RN64(x/h)) (pin P1); x == 0 gives 0.
// Returns whether the exact division is needed (also for non-finite x).
__device__ __forceinline__ bool gs_bin_floor_f32(float x, float ihf, int& k) {
  const float t = __fmul_rn(x, ihf);
  const float fl = floorf(t);
  const float fr = __fsub_rn(t, fl);
  const float eps = __fmaf_rn(fabsf(t), 0x1p-20f, 0x1p-23f);  // a margin, not a result
  k = __float2int_rz(fl);
  return !((fr > eps && fr < __fsub_rn(1.0f, eps) && fabsf(t) < 0x1p22f) || x == 0.0f);
}

// The binning front of one point: cell key per coordinate (box-relative), the linear index
// within the frame, fixed-point offsets q = RN(RN(x - RN(k*h)) * 2^F) (== gs_fixq).
template <int D, typename T>
struct BinPt {
  uint32_t loc;    // frame-local dense grid index (valid when ok)
  uint32_t dloc;   // index within the frame's data box (dense tables)
  bool ok, miss, nonfinite;
  long long q[D];
};

struct BinGeo {
  double h, inv_h, scale, magic;
  float ihf;
  bool f32fast, magic_ok;
  int kmin32[GS_DMAX];
  double kminD[GS_DMAX];
  uint32_t span[GS_DMAX], strd[GS_DMAX], dstrd[GS_DMAX];
};

template <int D, typename T>
__device__ __forceinline__ void bin_point(const T* xc, int64_t pl, const GsImg& im,
                                          const BinGeo& g, BinPt<D, T>& o) {
  double fl[D], xs[D];
  int rel[D];
  bool slow = false;
  if constexpr (sizeof(T) == 4) {
    if (g.f32fast) {
#pragma unroll
      for (int c = 0; c < D; ++c) {
        int k;
        slow |= gs_bin_floor_f32(xc[c], g.ihf, k);
        rel[c] = k - g.kmin32[c];
        fl[c] = (double)k;
        xs[c] = (double)xc[c];
      }
    } else {
      slow = true;
#pragma unroll
      for (int c = 0; c < D; ++c) xs[c] = (double)xc[c];
    }
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xs[c] = gs_feature<T, D>(xc, c, pl, im);
      slow |= gs_bin_floor(xs[c], g.inv_h, fl[c]);
      rel[c] = __double2int_rz(__dsub_rn(fl[c], g.kminD[c]));
    }
  }
  o.nonfinite = false;
  if (slow) {  // rare: the exact IEEE quotient (and the non-finite check) for every coordinate
#pragma unroll
    for (int c = 0; c < D; ++c) {
      o.nonfinite |= !isfinite(xs[c]);
      fl[c] = floor(gs_ddiv_slow(xs[c], g.h));
      const double r = __dsub_rn(fl[c], g.kminD[c]);
      rel[c] = (r > -4.0 && r < 2147483647.0) ? __double2int_rz(r) : -4;
    }
  }
  bool bad = o.nonfinite;
  uint32_t loc = 0, dloc = 0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const uint32_t dr = (uint32_t)(rel[c] - GS_APRON);
    bad |= dr >= g.span[c];
    loc += (uint32_t)rel[c] * g.strd[c];
    dloc += dr * g.dstrd[c];
    const double d = __dsub_rn(xs[c], __dmul_rn(fl[c], g.h));
    const double v = __dmul_rn(d, g.scale);
    // RN to an integer: the 1.5*2^52 trick is exact for |v| < 2^51 (F keeps |q| below it
    // when n >= 513), else the conversion instruction
    o.q[c] = g.magic_ok ? __double_as_longlong(__dadd_rn(v, g.magic)) - __double_as_longlong(g.magic)
                        : __double2ll_rn(v);
  }
  o.ok = !bad;
  o.miss = bad && !o.nonfinite;
  o.loc = loc;
  o.dloc = dloc;
}

// Warp aggregation over runs of equal keys (pixel-ordered images put most of a warp into 1-4
// runs): a run's sums reduce to its first lane with REDUX before any atomic.  Runs come from
// one shuffle + ballot (MATCH.ANY costs 2 cycles per distinct key).  A warp of many runs
// (shuffled clouds, noisy backgrounds) skips it.  Returns whether this lane carries atomics
// and its count.
template <int D>
__device__ __forceinline__ bool warp_runs(uint32_t key, bool act, long long* q, bool two_piece,
                                          uint32_t& my_cnt) {
  const unsigned lane = threadIdx.x & 31;
  const uint32_t prev = __shfl_up_sync(kFull, key, 1);
  const bool head = lane == 0 || key != prev;
  const unsigned heads = __ballot_sync(kFull, head);
  my_cnt = 1;
  if (__popc(heads) > kAggRuns) return act;
  const unsigned upto = heads & (0xffffffffu >> (31 - lane));    // heads <= lane
  const unsigned after = heads & ~(0xffffffffu >> (31 - lane));  // heads > lane
  const int s = 31 - __clz(upto);
  const int e = after ? __ffs(after) - 1 : 32;
  const unsigned gm = (e == 32 ? 0xffffffffu : ((1u << e) - 1u)) & ~((1u << s) - 1u);
  my_cnt = (uint32_t)__popc(gm);
  unsigned rem = heads;
  while (rem) {
    const int ld = __ffs(rem) - 1;
    rem &= rem - 1u;
    if (ld == s) {
      if (two_piece) {  // per-point |q| <= 2^51: 26-bit unsigned + signed high piece
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const long long u = q[c];
          const unsigned long long s0 = __reduce_add_sync(gm, (unsigned)(u & 0x3ffffff));
          const long long s1 = __reduce_add_sync(gm, (int)(u >> 26));
          q[c] = (long long)s0 + s1 * 67108864ll;
        }
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const unsigned long long u = (unsigned long long)q[c];
          const unsigned long long s0 = __reduce_add_sync(gm, (unsigned)(u & 0x3ffffffu));
          const unsigned long long s1 = __reduce_add_sync(gm, (unsigned)((u >> 26) & 0x3ffffffu));
          const unsigned long long s2 = __reduce_add_sync(gm, (unsigned)(u >> 52));
          q[c] = (long long)(s0 + (s1 << 26) + (s2 << 52));
        }
      }
    }
  }
  return act && head;  // only the run's first lane carries the run's sums
}

template <int D, typename T>
__global__ void __launch_bounds__(kBinThreads, 1)
    k_bin(const T* __restrict__ pts, int64_t ntot, const GsBox* __restrict__ pb,
          uint32_t* __restrict__ cnt, unsigned long long* __restrict__ qs, void* __restrict__ slot,
          int* err, int img_w, int predicted, int max_reps, int hash_rep_log2) {
  constexpr int RC = gs_raw_cols<T, D>();
  constexpr uint32_t EMPTY = 0xffffffffu;
  const int64_t per = (ntot + gridDim.x - 1) / gridDim.x;
  const int64_t p0 = (int64_t)blockIdx.x * per;
  const int64_t p1 = min(ntot, p0 + per);
  __shared__ GsBox b;
  __shared__ int s_err;
  if (threadIdx.x == 0) {
    s_err = *err;
    b = *pb;
  }
  __syncthreads();
  if (s_err & GS_ERR_SKIP) return;  // non-finite input / box beyond the grid: nothing to bin
  extern __shared__ __align__(16) unsigned char smem[];
  const unsigned lane = threadIdx.x & 31;
  const GsImg im = gs_img(img_w, b.n);
  BinGeo g;
  g.h = b.h;
  g.inv_h = b.inv_h;
  g.scale = b.scale;
  g.magic = 0x1.8p52;
  // per-point |q| <= h*2^F < 2^(ilogb(h)+1+F): <= 2^51 (n >= 513 points per frame) keeps the
  // RN-to-integer trick exact and lets a 32-lane sum split into two 32-bit pieces
  const bool two_piece = ilogb(b.h) + 1 + b.F <= 51;
  g.magic_ok = two_piece;
  g.ihf = __double2float_rn(b.inv_h);
  g.f32fast = true;
  uint32_t vd = 1;
#pragma unroll
  for (int c = D - 1; c >= 0; --c) {
    g.kminD[c] = (double)b.kmin[c];
    g.f32fast &= b.kmin[c] > -(1ll << 30) && b.kmin[c] < (1ll << 30);
    g.kmin32[c] = (int)b.kmin[c];
    g.span[c] = (uint32_t)(b.ext[c] - 2 * GS_APRON);
    g.strd[c] = (uint32_t)b.stride[c];
    g.dstrd[c] = vd;
    vd *= g.span[c];
  }
  const uint32_t vf = (uint32_t)b.vol_frame;
  const bool s16 = b.vol_frame <= 65536;
  uint16_t* slot16 = (uint16_t*)slot;
  uint32_t* slot32 = (uint32_t*)slot;
  const int errbit_box = predicted ? 128 : 2;
  // table plan: dense data box (with replicas) when it fits, else the hash table
  constexpr int EB = 4 + 8 * D;  // count + D x (lo, hi)
  const bool dense = (int64_t)vd * EB <= kBinSmemBytes;
  const int reps = dense ? max(1, min(max_reps, (int)(kBinSmemBytes / ((int64_t)vd * EB)))) : 1;
  const int rep_log2 = dense ? 0 : hash_rep_log2;
  const int TBL = dense ? (int)vd * reps : ((kBinSmemBytes / (EB + 4)) & ~31);
  unsigned* tc = (unsigned*)smem;                  // TBL counts
  unsigned* tlo = tc + TBL;                        // D x TBL low words
  unsigned* thi = tlo + (size_t)D * TBL;           // D x TBL high words
  uint32_t* tk = thi + (size_t)D * TBL;            // TBL keys (hash)
  for (int j = threadIdx.x; j < TBL; j += blockDim.x) {
    tc[j] = 0u;
#pragma unroll
    for (int c = 0; c < D; ++c) tlo[c * TBL + j] = thi[c * TBL + j] = 0u;
    if (!dense) tk[j] = EMPTY;
  }
  __syncthreads();
  bool saw_miss = false, saw_nan = false;
  // segments: dense tables hold one frame, so the range is cut at frame boundaries
  int64_t s0 = p0;
  while (s0 < p1) {
    const int64_t fr = s0 / b.n;
    const int64_t s1 = dense ? min(p1, (fr + 1) * b.n) : p1;
    const uint32_t fbase = (uint32_t)(fr * b.vol_frame);
    // frame tracking inside a hash segment (several frames)
    int64_t hfr = (s0 + threadIdx.x) / b.n, hfr_end = (hfr + 1) * b.n;
    uint32_t hbase = (uint32_t)(hfr * b.vol_frame);
    T xn[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) xn[c] = (s0 + threadIdx.x < s1) ? pts[(s0 + threadIdx.x) * RC + c] : T(0);
    // warp-uniform trip count so every lane takes part in the warp aggregation; the next
    // round's coordinates are loaded before this round is processed
    for (int64_t pr = s0; pr < s1; pr += blockDim.x) {
      const int64_t p = pr + threadIdx.x;
      const bool valid = p < s1;
      T xc[RC];
#pragma unroll
      for (int c = 0; c < RC; ++c) xc[c] = xn[c];
      const int64_t pn = p + blockDim.x;
#pragma unroll
      for (int c = 0; c < RC; ++c) xn[c] = pn < s1 ? pts[pn * RC + c] : T(0);
      if (!dense) {
        while (p >= hfr_end) {
          ++hfr;
          hfr_end += b.n;
          hbase += vf;
        }
      }
      const uint32_t base = dense ? fbase : hbase;
      BinPt<D, T> o;
      bin_point<D, T>(xc, (sizeof(T) == 1 && D > 3) ? p - (dense ? fr : hfr) * b.n : 0, im, g, o);
      uint32_t key = EMPTY;
      if (valid) {
        if (o.ok) {
          if (s16) slot16[p] = (uint16_t)o.loc;
          else slot32[p] = base + o.loc;
          key = dense ? o.dloc : base + o.loc;
        } else {
          saw_nan |= o.nonfinite;
          saw_miss |= o.miss;
        }
      }
      uint32_t my_cnt;
      const bool act = warp_runs<D>(key, key != EMPTY, o.q, two_piece, my_cnt);
      const unsigned am = __ballot_sync(kFull, act);
      if (dense) {
        if (act) {
          const uint32_t e = (lane % (unsigned)reps) * vd + key;
          atomicAdd(&tc[e], my_cnt);
#pragma unroll
          for (int c = 0; c < D; ++c)
            smem_add64(&tlo[c * TBL + e], &thi[c * TBL + e], (unsigned long long)o.q[c]);
        }
      } else if (act) {
        // predicated probe loop, then the active lanes reconverge before the atomics (an
        // early-exit loop let the compiler replay the atomic sequence once per exit group)
        const uint32_t tkey = (key << rep_log2) | (lane & ((1u << rep_log2) - 1u));
        uint32_t hsh = __umulhi(tkey * 2654435761u, (unsigned)TBL);
        int hit = -1;
#pragma unroll
        for (int probe = 0; probe < kBinProbes; ++probe) {
          if (hit < 0) {
            uint32_t k = tk[hsh];
            if (k == EMPTY) k = atomicCAS(&tk[hsh], EMPTY, tkey);
            if (k == EMPTY || k == tkey) hit = (int)hsh;
            hsh = (hsh + 1 == (unsigned)TBL) ? 0u : hsh + 1;
          }
        }
        __syncwarp(am);
        if (hit >= 0) {
          atomicAdd(&tc[hit], my_cnt);
#pragma unroll
          for (int c = 0; c < D; ++c)
            smem_add64(&tlo[c * TBL + hit], &thi[c * TBL + hit], (unsigned long long)o.q[c]);
        } else {
          atomicAdd(&cnt[key], my_cnt);
#pragma unroll
          for (int c = 0; c < D; ++c) atomicAdd(&qs[(size_t)key * D + c], (unsigned long long)o.q[c]);
        }
      }
    }
    __syncthreads();
    if (dense) {  // flush this frame's table (replicas summed) and leave it zeroed
      for (uint32_t j = threadIdx.x; j < vd; j += blockDim.x) {
        unsigned cn = 0;
        for (int r = 0; r < reps; ++r) cn += tc[r * vd + j];
        if (!cn) continue;
        uint32_t L = fbase, rem = j;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const uint32_t dr = rem / g.dstrd[c];
          rem -= dr * g.dstrd[c];
          L += (dr + GS_APRON) * g.strd[c];
        }
        atomicAdd(&cnt[L], cn);
        for (int r = 0; r < reps; ++r) tc[r * vd + j] = 0u;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          unsigned long long sq = 0ull;
          for (int r = 0; r < reps; ++r) {
            const uint32_t e = r * vd + j;
            sq += ((unsigned long long)thi[c * TBL + e] << 32) | tlo[c * TBL + e];
            tlo[c * TBL + e] = thi[c * TBL + e] = 0u;
          }
          atomicAdd(&qs[(size_t)L * D + c], sq);
        }
      }
      __syncthreads();
    }
    s0 = s1;
  }
  if (saw_nan) atomicOr(err, 1);
  if (saw_miss) atomicOr(err, errbit_box);
  if (!dense) {
    for (int j = threadIdx.x; j < TBL; j += blockDim.x) {
      const uint32_t key = tk[j];
      if (key == EMPTY) continue;
      const int64_t L = key >> rep_log2;
      atomicAdd(&cnt[L], tc[j]);
#pragma unroll
      for (int c = 0; c < D; ++c)
        atomicAdd(&qs[L * D + c], ((unsigned long long)thi[c * TBL + j] << 32) | tlo[c * TBL + j]);
    }
  }
}


// Predicted key box (no bounds pass): the box of the previous run of this shape.
__global__ void k_box_set(GsBox b, GsBox* __restrict__ out, unsigned* epoch) {
  *out = b;
  *epoch += 1u;
}

// ---------------------------------------------------------------- K3: compaction by scan
// The dense grid is in lexicographic order, so scanning its occupancy yields the cell list
// already sorted: no occupied list, no sort, no host round trip for m0.
constexpr int kOccPer = 2;                // cells per thread
constexpr int kOccTile = 256 * kOccPer;   // cells per tile (256 threads)

__device__ __forceinline__ int block_excl_scan_256(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < 8 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int y = __shfl_up_sync(kFull, t, o);
      if (lane >= o) t += y;
    }
    if (lane < 8) sh[lane] = t;
  }
  __syncthreads();
  const int excl = x - v + (w > 0 ? sh[w - 1] : 0);
  *total = sh[7];
  __syncthreads();
  return excl;
}

// Single pass (decoupled look-back): tiles are taken in ticket order; each publishes its
// occupied-cell count, then sums its predecessors' counts (a warp reads 32 flags at a time)
// until one that already carries its inclusive prefix.  Flags are tagged with the run epoch,
// so the flag array is never cleared.  Per occupied cell: lex-ordered cell list, centroid from
// the fixed-point sums, clean-grid restore (cnt = qs = 0), idx = slot; per frame: the first
// cell index (ifirst[nframes] = m0).
__device__ __forceinline__ unsigned long long occ_flag(unsigned epoch, unsigned st, unsigned v) {
  return ((unsigned long long)epoch << 32) | ((unsigned long long)st << 30) | v;
}

__global__ void __launch_bounds__(256) k_occ(
    const GsBox* __restrict__ pb, const unsigned* __restrict__ epoch_p,
    unsigned long long* tflag, unsigned* ticket, unsigned* m0_out, uint32_t* __restrict__ cnt,
    unsigned long long* __restrict__ qs, uint32_t* __restrict__ ckey,
    uint32_t* __restrict__ ccnt, double* __restrict__ S, int32_t* __restrict__ idx,
    int32_t* __restrict__ root, uint32_t* __restrict__ initkey, int32_t* __restrict__ ifirst,
    const int* __restrict__ err, long long* __restrict__ xsum = nullptr) {
  // xsum != null: export mode (a shard's partial cells for the multi-GPU exchange): keys,
  // counts and the raw fixed-point sums, no centroids, no index / root / label entries
  if (*err & GS_ERR_SKIP) return;
  __shared__ int sh[8];
  __shared__ GsBox b;
  __shared__ int s_tile, s_excl;
  if (threadIdx.x == 0) b = *pb;
  const unsigned E = *epoch_p;
  __syncthreads();
  const int64_t V = b.vol_total, VF = b.vol_frame;
  const int64_t ntiles = (V + kOccTile - 1) / kOccTile;
  const int lane = threadIdx.x & 31;
  for (;;) {
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
    __syncthreads();
    const int64_t t = s_tile;
    if (t >= ntiles) break;
    const int64_t base = t * kOccTile + (int64_t)threadIdx.x * kOccPer;
    uint32_t c8[kOccPer];
    int c = 0;
#pragma unroll
    for (int k = 0; k < kOccPer; ++k) {
      c8[k] = (base + k < V) ? cnt[base + k] : 0u;
      c += c8[k] != 0u;
    }
    int total;
    const int excl = block_excl_scan_256(c, sh, &total);
    if (threadIdx.x < 32) {  // publish, then look back (warp-wide)
      if (t == 0) {
        if (lane == 0) {
          atomicExch(&tflag[0], occ_flag(E, 2u, (unsigned)total));
          s_excl = 0;
        }
      } else {
        if (lane == 0) atomicExch(&tflag[t], occ_flag(E, 1u, (unsigned)total));
        int prefix = 0;
        int64_t hi = t - 1;  // flags [hi-31, hi] are examined per round
        for (;;) {
          const int64_t j = hi - lane;
          unsigned long long fw = 0ull;
          unsigned st = 3u;  // 3: beyond tile 0 (treated as an inclusive zero)
          if (j >= 0) {
            do {
              fw = *(volatile unsigned long long*)&tflag[j];
              st = ((unsigned)(fw >> 32) == E) ? (unsigned)(fw >> 30) & 3u : 0u;
            } while (st == 0u);
          }
          // the nearest lane (lowest index = highest tile) holding an inclusive prefix
          const unsigned incl = __ballot_sync(kFull, st >= 2u);
          const int stop = incl ? __ffs(incl) - 1 : 32;
          int v = (lane <= stop && st != 3u) ? (int)(fw & 0x3fffffffu) : 0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
          prefix += v;
          if (incl) break;
          hi -= 32;
        }
        if (lane == 0) {
          atomicExch(&tflag[t], occ_flag(E, 2u, (unsigned)(prefix + total)));
          s_excl = prefix;
        }
      }
    }
    __syncthreads();
    int pos = s_excl + excl;
    if (t == ntiles - 1 && threadIdx.x == 0) {
      *m0_out = (unsigned)(s_excl + total);
      ifirst[b.nframes] = s_excl + total;
    }
    int64_t f = base / VF, r = base - f * VF;
#pragma unroll
    for (int k = 0; k < kOccPer; ++k) {
      const int64_t L = base + k;
      if (L < V && r == 0) ifirst[f] = pos;  // first cell index of frame f
      if (++r == VF) {
        r = 0;
        ++f;
      }
      if (c8[k] == 0u) continue;
      for (int q = 0; q < b.d; ++q) {
        const long long sq = (long long)qs[L * b.d + q];
        if (xsum)
          xsum[(int64_t)pos * b.d + q] = sq;
        else
          S[(int64_t)pos * b.d + q] =
              gs_fix_centroid(gs_key_of(b, L, q), sq, c8[k], b.h, b.inv_scale);
        qs[L * b.d + q] = 0ull;
      }
      cnt[L] = 0u;
      ckey[pos] = (uint32_t)L;
      ccnt[pos] = c8[k];
      if (!xsum) {
        idx[L] = pos;
        root[pos] = pos;
        initkey[pos] = (uint32_t)L;
      }
      ++pos;
    }
    __syncthreads();  // s_tile / s_excl are rewritten by the next round
  }
}

// Multi-GPU (one cloud over R ranks): accumulate every rank's partial cells into the dense
// grid.  Counts and fixed-point sums are integers, so the merged grid equals the one a single
// GPU binning all points would build, bit for bit, in any order.
__global__ void k_scatter_partials(int64_t m, int d, const uint32_t* __restrict__ keys,
                                   const uint32_t* __restrict__ counts,
                                   const long long* __restrict__ sums, uint32_t* __restrict__ cnt,
                                   unsigned long long* __restrict__ qs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t L = keys[i];
    atomicAdd(&cnt[L], counts[i]);
    for (int c = 0; c < d; ++c) atomicAdd(&qs[L * d + c], (unsigned long long)sums[i * d + c]);
  }
}

// ---------------------------------------------------------------- K5: rehome
// New key floor(S/h) per cell (SPEC.md:120(d)), per-frame `changed` (SPEC.md:120(e)) and max
// sweep displacement.  Frozen frames keep their keys.
__global__ void k_rehome(int m, GsBox b, const uint32_t* __restrict__ ckey,
                         const double* __restrict__ S0, const double* __restrict__ S1,
                         const int32_t* __restrict__ fdone, uint32_t* __restrict__ nkey,
                         uint32_t* __restrict__ vals, int32_t* __restrict__ fchanged,
                         unsigned long long* __restrict__ fdisp, int* err) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t L = ckey[i];
  const int64_t f = L / b.vol_frame;
  vals[i] = (uint32_t)i;
  if (fdone[f]) {
    nkey[i] = (uint32_t)L;
    return;
  }
  int64_t Ln = f * b.vol_frame;
  bool changed = false, bad = false;
  double acc = 0.0;
  for (int c = 0; c < b.d; ++c) {
    const double s1 = S1[(int64_t)i * b.d + c], s0 = S0[(int64_t)i * b.d + c];
    const int64_t rel = gs_grid_coord(s1, b.h, b.inv_h) - b.kmin[c];
    bad |= (rel < 1) | (rel > b.ext[c] - 2);
    Ln += rel * b.stride[c];
    changed |= __double_as_longlong(s1) != __double_as_longlong(s0);
    const double t = __dsub_rn(s1, s0);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  if (bad) {
    atomicOr(err, 4);
    Ln = L;
  }
  changed |= (Ln != L);
  if (changed) fchanged[f] = 1;
  atomicMax(&fdisp[f], (unsigned long long)__double_as_longlong(__dsqrt_rn(acc)));
  nkey[i] = (uint32_t)Ln;
}

// segment heads of the (new key, old rank)-sorted pairs
__global__ void k_heads(int m, const uint32_t* __restrict__ skey, int32_t* __restrict__ head) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  head[j] = (j == 0 || skey[j] != skey[j - 1]) ? 1 : 0;
}

// parent map and segment starts from the inclusive scan of heads
__global__ void k_seg(int m, const int32_t* __restrict__ head, const int32_t* __restrict__ sid,
                      const uint32_t* __restrict__ sval, int32_t* __restrict__ parent,
                      int32_t* __restrict__ segstart) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int g = sid[j] - 1;
  parent[sval[j]] = g;
  if (head[j]) segstart[g] = j;
}

// merge_into folded in visit order (Eq. 3-4, pin P4): members of a segment are in increasing
// old rank because the sort is stable and ranks were fed in order.
// Ordered Eq. (3) fold of each new cell's members in visit order (pin P4), one thread per new
// cell: s = RN(RN(RN(a*s) + RN(w*S_i)) / tot) with the division from y = RN(1/tot) (Markstein,
// correctly rounded for integer tot; y does not depend on s, so it leaves the chain); an
// operand outside the theorem's range redoes the group with IEEE divisions.
template <int D>
__global__ void k_fold(int mnew, int m, const int32_t* __restrict__ segstart,
                       const uint32_t* __restrict__ skey, const uint32_t* __restrict__ sval,
                       const uint32_t* __restrict__ ccnt, const double* __restrict__ S1,
                       uint32_t* __restrict__ okey, uint32_t* __restrict__ ocnt,
                       double* __restrict__ oS) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= mnew) return;
  const int start = segstart[g];
  const int end = (g + 1 < mnew) ? segstart[g + 1] : m;
  const uint32_t i0 = sval[start];
  double s[D];
#pragma unroll
  for (int c = 0; c < D; ++c) s[c] = S1[(int64_t)i0 * D + c];
  uint64_t cnt = ccnt[i0];
  bool slow = false;
  // software-pipelined: the next member's index, count and row are loaded before this member
  // is folded (they do not depend on the fold), so only the fp64 chain is serial
  uint32_t in = start + 1 < end ? sval[start + 1] : 0u;
  uint64_t cin = start + 1 < end ? ccnt[in] : 0u;
  double Sn[D];
#pragma unroll
  for (int c = 0; c < D; ++c) Sn[c] = start + 1 < end ? S1[(int64_t)in * D + c] : 0.0;
  for (int j = start + 1; j < end; ++j) {
    const uint64_t ci = cin;
    double Si[D];
#pragma unroll
    for (int c = 0; c < D; ++c) Si[c] = Sn[c];
    if (j + 1 < end) {
      in = sval[j + 1];
      cin = ccnt[in];
#pragma unroll
      for (int c = 0; c < D; ++c) Sn[c] = S1[(int64_t)in * D + c];
    }
    const double a = (double)cnt, w = (double)ci, tot = (double)(cnt + ci);
    const double y = __drcp_rn(tot);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double num = __dadd_rn(__dmul_rn(a, s[c]), __dmul_rn(w, Si[c]));
      const double fa = fabs(num);
      slow |= !(fa < 0x1p+1000) || (fa < 0x1p-900 && num != 0.0);
      const double q0 = __dmul_rn(num, y);
      s[c] = __fma_rn(__fma_rn(-q0, tot, num), y, q0);
    }
    cnt += ci;
  }
  if (slow) {
    cnt = ccnt[i0];
#pragma unroll
    for (int c = 0; c < D; ++c) s[c] = S1[(int64_t)i0 * D + c];
    for (int j = start + 1; j < end; ++j) {
      const uint32_t i = sval[j];
      const uint64_t ci = ccnt[i];
      const double a = (double)cnt, w = (double)ci, tot = (double)(cnt + ci);
#pragma unroll
      for (int c = 0; c < D; ++c)
        s[c] = gs_ddiv_slow(__dadd_rn(__dmul_rn(a, s[c]), __dmul_rn(w, S1[(int64_t)i * D + c])),
                            tot);
      cnt += ci;
    }
  }
  okey[g] = skey[start];
  ocnt[g] = (uint32_t)cnt;
#pragma unroll
  for (int c = 0; c < D; ++c) oS[(int64_t)g * D + c] = s[c];
}

__global__ void k_idx_clear(int m, const uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) idx[key[i]] = -1;
}

__global__ void k_idx_set(int m, const uint32_t* __restrict__ key, int32_t* __restrict__ idx) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) idx[key[i]] = i;
}

// has_converged per frame: fadj[f] = 1 if some cell of f has another
// active cell in its 1-neighbourhood.  D <= 6: batched probes from a shared offset table.
template <int D>
__global__ void k_adjacent(int m, GsBox b, int K, const uint32_t* __restrict__ key,
                           const int32_t* __restrict__ idx, const int32_t* __restrict__ fdone,
                           int32_t* __restrict__ fadj) {
  if constexpr (D <= 6) {
    constexpr int KMAX = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : D == 5 ? 243 : 729;
    constexpr int B = KMAX < 27 ? KMAX : 27;
    __shared__ int offs[KMAX];
    for (int t = threadIdx.x; t < KMAX; t += blockDim.x) {
      int r = t;
      int64_t off = 0;
      for (int c = D - 1; c >= 0; --c) {
        off += (int64_t)(r % 3 - 1) * b.stride[c];
        r /= 3;
      }
      offs[t] = (int)off;
    }
    __syncthreads();
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t L = key[i];
    const int64_t f = L / b.vol_frame;
    if (fdone[f]) return;
    for (int t0 = 0; t0 < KMAX; t0 += B) {
      int hit = 0;
#pragma unroll
      for (int u = 0; u < B; ++u)
        hit |= (t0 + u != (KMAX - 1) / 2) & (__ldg(&idx[L + offs[t0 + u]]) >= 0);
      if (hit) {
        fadj[f] = 1;
        return;
      }
    }
  } else {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t L = key[i];
    const int64_t f = L / b.vol_frame;
    if (fdone[f]) return;
    GsNbrOdometer od;
    od.init(b);
    for (int t = 0; t < K; ++t) {
      if (od.off != 0 && idx[L + od.off] >= 0) {
        fadj[f] = 1;
        return;
      }
      od.next(b);
    }
  }
}

// member union H (Eq. 4) as a composed parent map: root[c0] <- parent[root[c0]]
__global__ void k_compose(int m0, const int32_t* __restrict__ parent, int32_t* __restrict__ root) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m0) root[i] = parent[root[i]];
}

// K7: labels[p] = lab[cell of p].  Frames are blockIdx.y-strided, so a point's frame base is
// known without a division; u16 slots are read 8 at a time (16-byte loads).  Block (0, 0) also
// hands the run's control block to the host: it stores the words into mapped pinned memory (no
// copy node, ~12 us per run on the graph path) and then re-zeroes the part every run starts
// from zero, so the next run needs no memset node either.
__global__ void __launch_bounds__(256) k_label(int64_t n, int64_t nf, const void* __restrict__ slot,
                                               const GsBox* __restrict__ pb,
                                               const int32_t* __restrict__ lab,
                                               int32_t* __restrict__ labels,
                                               unsigned* __restrict__ ctl, unsigned* ctl_host,
                                               int ctl_words, int zero_words) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && ctl_host) {
    for (int w = threadIdx.x; w < ctl_words; w += blockDim.x) ctl_host[w] = ctl[w];
    __syncthreads();
    for (int w = threadIdx.x; w < zero_words; w += blockDim.x) ctl[w] = 0u;
  }
  const int64_t vf = pb->vol_frame;
  const bool s16 = vf <= 65536;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  // u16 slots: a lane takes 4 consecutive points (8-byte slot load, 16-byte label store), so a
  // warp instruction reads 256 contiguous bytes and writes 512 (whole lines: also for labels
  // written straight into pinned host memory)
  const bool vec = s16 && (n % 4) == 0 && (((uintptr_t)slot | (uintptr_t)labels) & 15) == 0;
  for (int64_t f = blockIdx.y; f < nf; f += gridDim.y) {
    const int64_t p0 = f * n;
    const uint32_t fbase = (uint32_t)(f * vf);
    if (vec) {
      const uint2* s4 = reinterpret_cast<const uint2*>((const uint16_t*)slot + p0);
      int4* o4 = reinterpret_cast<int4*>(labels + p0);
      for (int64_t i = tid; i < n / 4; i += nth) {
        const uint2 w = s4[i];
        o4[i] = make_int4(__ldg(&lab[fbase + (w.x & 0xffffu)]), __ldg(&lab[fbase + (w.x >> 16)]),
                          __ldg(&lab[fbase + (w.y & 0xffffu)]), __ldg(&lab[fbase + (w.y >> 16)]));
      }
    } else {
      for (int64_t i = tid; i < n; i += nth)
        labels[p0 + i] = __ldg(&lab[gs_slot_cell(slot, s16, p0 + i, fbase)]);
    }
  }
}

// Segmentation render: a segment's colour is its centroid's first three
// components times 255, rounded half-up, clamped to 0..255 (packed r | g<<8 | b<<16)
__global__ void k_segment_colours(int64_t k, int d, const double* __restrict__ cent,
                                  uint32_t* __restrict__ rgb) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= k) return;
  uint32_t packed = 0;
  for (int c = 0; c < 3; ++c) {
    double v = floor(__dadd_rn(__dmul_rn(cent[g * d + c], 255.0), 0.5));
    v = fmin(fmax(v, 0.0), 255.0);
    packed |= (uint32_t)v << (8 * c);
  }
  rgb[g] = packed;
}

// every pixel -> its segment's colour (label = lab[slot[p]], as K7)
__global__ void __launch_bounds__(256) k_render(int64_t n, const void* __restrict__ slot,
                                                int64_t frame, const GsBox* __restrict__ pb,
                                                const int32_t* __restrict__ lab,
                                                const uint32_t* __restrict__ rgb,
                                                uint8_t* __restrict__ out) {
  const bool s16 = pb->vol_frame <= 65536;
  const uint32_t fbase = (uint32_t)(frame * pb->vol_frame);
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = rgb[lab[gs_slot_cell(slot, s16, frame * n + p, fbase)]];
    out[3 * p] = (uint8_t)(v & 0xffu);
    out[3 * p + 1] = (uint8_t)((v >> 8) & 0xffu);
    out[3 * p + 2] = (uint8_t)((v >> 16) & 0xffu);
  }
}

// test hook: rank of every point's initial cell
__global__ void k_slot_rank(int64_t ntot, const void* __restrict__ slot,
                            const GsBox* __restrict__ pb, const int32_t* __restrict__ idx,
                            int64_t* __restrict__ out) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < ntot) out[p] = idx[gs_slot_cell(slot, pb->vol_frame <= 65536, p, 0u)];
}

}  // namespace gs
