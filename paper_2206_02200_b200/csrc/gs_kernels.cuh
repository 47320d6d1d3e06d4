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

#include <cmath>
#include <cstring>

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
// 64-bit shared add; atomicAdd(u64) compiles to a CAS loop).  An entry is EW = 1 + 2D words
// [count, lo_0, hi_0, ...]: an odd word stride, so random entries spread over the banks.
//
// Predicted box (`predicted` != 0): the key box is the one the previous run of this shape used
// (no bounds pass); a point outside it sets err bit 128 (the host clears the grid and reruns
// with the bounds pass) and a non-finite coordinate sets bit 1.
#ifndef GS_BIN_THREADS
#define GS_BIN_THREADS 1024  // (experiments override it at build time)
#endif
#ifndef GS_BIN_CTAS
#define GS_BIN_CTAS 1        // K2 CTAs per SM
#endif
constexpr int kBinThreads = GS_BIN_THREADS;
constexpr int kBinCtas = GS_BIN_CTAS;
constexpr int kBinProbes = 4;  // hash probe budget before the point takes the global atomics
constexpr int kAggRuns = 4;    // warp aggregation when the warp's keys form <= this many runs
constexpr int kBinSmemBytes = (kBinCtas == 1 ? 224 : 112) * 1024;

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

// fp32 inputs: the same floor from fp32 arithmetic, with no FRND/F2I (16 lanes/clk/SM on
// sm_100, measured: profiles/r2_microbench_conv.txt).  u = RN(x*ihf + C) with C = 1.5*2^23 - kmin
// is rint(v) - kmin + 1.5*2^23 for the exact product v = x*ihf (ihf = RN32(1/h), |v - x/h| <=
// |x/h| 2^-23.9) while |v - kmin| < 2^22; nr = C - u = -rint(v) exactly; d = RN(v - rint(v)).
// When |d| > |rint(v)| 2^-20, x/h lies on v's side of the integer rint(v), so floor(x/h) ==
// floor(RN64(x/h)) == rint(v) - (d < 0) (pin P1); x == +-0 gives 0.  The test uses the launch
// constant thr = (max |key of the box| + 2) * 2^-20 >= |rint(v)| 2^-20 for every point in or
// next to the box (one compare instead of a multiply and two compares); a point farther out
// may take a key off by one, which is still outside the box and flagged.  Outside the magic
// range the decoded key lies beyond the box (the host enables this path only for extents
// < 2^21), so the point is flagged, never mis-binned.  Returns the key relative to the box
// origin.
__device__ __forceinline__ int gs_bin_rel_f32(float x, float ihf, float C, float thr, bool& fine) {
  const float u = __fmaf_rn(x, ihf, C);
  const float nr = __fsub_rn(C, u);
  const float d = __fmaf_rn(x, ihf, nr);  // (-0 + +0 = +0: x == -0 gives key 0)
  fine = (fabsf(d) > thr) | (x == 0.0f);
  return (__float_as_int(u) - 0x4B400000) + (__float_as_int(d) >> 31);
}

// Launch geometry of K2, computed on the host from the key box (kernel parameters live in the
// constant bank: no registers for the per-dimension constants).
struct BinParams {
  double h, inv_h, scale, Mq;  // Mq = 1.5*2^(52-F): RN(d + Mq) - Mq = RN to the 2^-F grid
  long long Mbits;             // bits of Mq: table sums carry count * Mbits, removed at flush
  long long n, vol_frame;
  float ihf, thr;               // thr: fp32 key fineness threshold (gs_bin_rel_f32)
  float s2F, xmin;              // X path: 2^F, and the least |x| whose x*2^F is an integer
  int magic_ok, two_piece, f32fast, xpath, dense, reps, TBL, rep_log2, s16, predicted;
  uint32_t vd;                 // cells of a frame's data box
  float Cf[GS_DMAX];           // 1.5*2^23 - kmin (fp32 fast key)
  int kmin32[GS_DMAX];
  double kminD[GS_DMAX];
  uint32_t span[GS_DMAX], strd[GS_DMAX], dstrd[GS_DMAX];
};

template <int D>
inline BinParams make_bin_params(const GsBox& b, int max_reps, int hash_rep_log2, int predicted) {
  BinParams P;
  memset(&P, 0, sizeof(P));
  P.h = b.h;
  P.inv_h = b.inv_h;
  P.scale = b.scale;
  P.n = b.n;
  P.vol_frame = b.vol_frame;
  P.two_piece = (std::ilogb(b.h) + 1 + b.F) <= 51;
  P.magic_ok = P.two_piece;
  P.Mq = std::ldexp(1.5, 52 - b.F);
  std::memcpy(&P.Mbits, &P.Mq, 8);
  P.ihf = (float)b.inv_h;
  P.f32fast = P.magic_ok;
  uint32_t vd = 1;
  for (int c = D - 1; c >= 0; --c) {
    P.kminD[c] = (double)b.kmin[c];
    P.f32fast &= b.kmin[c] > -(1ll << 21) && b.kmin[c] < (1ll << 21) && b.ext[c] < (1ll << 21);
    P.kmin32[c] = (int)b.kmin[c];
    P.Cf[c] = 12582912.0f - (float)P.kmin32[c];
    P.span[c] = (uint32_t)(b.ext[c] - 2 * GS_APRON);
    P.strd[c] = (uint32_t)b.stride[c];
    P.dstrd[c] = vd;
    vd *= P.span[c];
  }
  P.vd = vd;
  int64_t kmax = 0;
  for (int c = 0; c < D; ++c)
    kmax = std::max<int64_t>(kmax, std::max(std::llabs(b.kmin[c]), std::llabs(b.kmin[c] + b.ext[c])));
  P.thr = std::ldexp((float)(kmax + 2), -20);
  P.s16 = b.vol_frame <= 65536;
  // dense data box (with replicas) when it fits and the frame's cells fit u16 slots
  constexpr int EW = 1 + 2 * D;
  P.dense = P.s16 && (int64_t)vd * EW * 4 <= kBinSmemBytes;
  P.reps = P.dense ? std::max(1, std::min(max_reps, (int)(kBinSmemBytes / ((int64_t)vd * EW * 4)))) : 1;
  P.TBL = P.dense ? (int)vd * P.reps : ((kBinSmemBytes / (EW * 4 + 4)) & ~31);
  // The fp32 fast path sums X = x*2^F (an integer for |x| >= 2^(23-F)) instead of q: with
  // c = RN(k*h), RN(x - c) is exact (Sterbenz for |k| >= 1 and for k = -1, |x| >= h/2; k = 0
  // trivially; k = -1, |x| < h/2 because x is a multiple of 2^-F >= ulp(h)/2), so q =
  // RHE((x - c)*2^F) = X - Cr with Cr = RHE(c*2^F), unless c*2^F has fraction exactly 1/2 (a
  // tie: the path is refused for the whole box).  The table sums X; the flush takes count*Cr.
  // |X| < 2^52 keeps the two-piece warp reduction and F2I exact.
  if (P.f32fast && P.dense) {
    const int F = b.F;
    bool ok = F <= 53 - std::ilogb(b.h) && F <= 120 && F >= -100;
    ok = ok && std::ldexp((double)(kmax + 2) * b.h, F) < 0x1p52;
    int64_t tot = 0;
    for (int c = 0; c < D; ++c) tot += b.ext[c];
    ok = ok && tot <= 65536;
    for (int c = 0; ok && c < D; ++c)
      for (int64_t k = b.kmin[c]; ok && k < b.kmin[c] + b.ext[c]; ++k) {
        const double C = std::ldexp((double)k * b.h, F);
        ok = C - std::floor(C) != 0.5;
      }
    P.xpath = ok;
    P.s2F = std::ldexp(1.0f, F);
    P.xmin = std::ldexp(1.0f, 23 - F);
  }
  P.rep_log2 = P.dense ? 0 : hash_rep_log2;
  P.predicted = predicted;
  return P;
}

// The binning front of one point: cell key per coordinate (box-relative), the linear index
// within the frame (loc) and within the frame's data box (dloc), and the fixed-point offsets
// q = RN(RN(x - RN(k*h)) * 2^F) (== gs_fixq) as w = q + Mbits when magic_ok (the 1.5*2^(52-F)
// trick: |q| <= 2^51), else q itself; XP (the fp32 X path of dense tables): w = X = x*2^F, and
// q = X - Cr (the table sums X, the flush takes count * Cr, bin_cr).  Returns 0 ok, 1 outside
// the box, 2 non-finite.

// X path: Cr = RHE(RN(k*h) * 2^F) of key k (q = X - Cr)
__device__ __forceinline__ long long bin_cr(int k, const BinParams& P) {
  return __double2ll_rn(__dmul_rn(__dmul_rn((double)k, P.h), P.scale));
}

template <int D, typename T, bool FAST, bool XP>
__device__ __forceinline__ int bin_point(const T* xc, int64_t pl, const GsImg& im,
                                         const BinParams& P, uint32_t& loc, uint32_t& dloc,
                                         long long* w) {
  int rel[D];
  if constexpr (XP) {  // the X path: w = x*2^F, no fp64 (see make_bin_params)
    bool fine = true;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      bool f;
      const float x = (float)xc[c];
      rel[c] = gs_bin_rel_f32(x, P.ihf, P.Cf[c], P.thr, f);
      fine &= f & ((fabsf(x) >= P.xmin) | (x == 0.0f));
      w[c] = __float2ll_rn(__fmul_rn(x, P.s2F));
    }
    bool nonfinite = false;
    if (!fine) {  // rare: the IEEE quotient, and w = q + Cr for an x that is not a multiple of 2^-F
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double x = (double)xc[c];
        nonfinite |= !isfinite(x);
        const double f = floor(gs_ddiv_slow(x, P.h));
        const double r = __dsub_rn(f, P.kminD[c]);
        rel[c] = (r > -4.0 && r < 2147483647.0) ? __double2int_rz(r) : -4;
        const double ck = __dmul_rn(f, P.h);
        w[c] = __double2ll_rn(__dmul_rn(__dsub_rn(x, ck), P.scale)) +
               __double2ll_rn(__dmul_rn(ck, P.scale));
      }
    }
    bool bad = false;
    uint32_t l = 0, dl = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const uint32_t dr = (uint32_t)(rel[c] - GS_APRON);
      bad |= dr >= P.span[c];
      l += (uint32_t)rel[c] * P.strd[c];
      dl += dr * P.dstrd[c];
    }
    loc = l;
    dloc = dl;
    return nonfinite ? 2 : bad ? 1 : 0;
  }
  double fl[D], xs[D];
  bool slow = false;
  if constexpr (FAST) {
    bool fine = true;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      bool f;
      rel[c] = gs_bin_rel_f32(xc[c], P.ihf, P.Cf[c], P.thr, f);
      fine &= f;
      fl[c] = (double)(rel[c] + P.kmin32[c]);
      xs[c] = (double)xc[c];
    }
    slow = !fine;
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      xs[c] = gs_feature<T, D>(xc, c, pl, im);
      slow |= gs_bin_floor(xs[c], P.inv_h, fl[c]);
      rel[c] = __double2int_rz(__dsub_rn(fl[c], P.kminD[c]));
    }
  }
  bool nonfinite = false;
  if (slow) {  // rare: the exact IEEE quotient (and the non-finite check) for every coordinate
#pragma unroll
    for (int c = 0; c < D; ++c) {
      nonfinite |= !isfinite(xs[c]);
      fl[c] = floor(gs_ddiv_slow(xs[c], P.h));
      const double r = __dsub_rn(fl[c], P.kminD[c]);
      rel[c] = (r > -4.0 && r < 2147483647.0) ? __double2int_rz(r) : -4;
    }
  }
  bool bad = false;
  uint32_t l = 0, dl = 0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const uint32_t dr = (uint32_t)(rel[c] - GS_APRON);
    bad |= dr >= P.span[c];
    l += (uint32_t)rel[c] * P.strd[c];
    dl += dr * P.dstrd[c];
    const double dd = __dsub_rn(xs[c], __dmul_rn(fl[c], P.h));
    if (FAST || P.magic_ok)  // (the fast key path is only taken with magic_ok)
      w[c] = __double_as_longlong(__dadd_rn(dd, P.Mq));
    else
      w[c] = __double2ll_rn(__dmul_rn(dd, P.scale));
  }
  loc = l;
  dloc = dl;
  return nonfinite ? 2 : bad ? 1 : 0;
}

// Warp aggregation over runs of equal keys (pixel-ordered images put most of a warp into 1-4
// runs): a run's sums reduce to its first lane with REDUX before any atomic.  Runs come from
// one shuffle + ballot (MATCH.ANY costs 2 cycles per distinct key).  A warp of many runs
// (shuffled clouds, noisy backgrounds) skips it.  w holds q + off per lane; the run head gets
// sum(q) + count * off.  Returns whether this lane carries atomics and its count.
template <int D>
__device__ __forceinline__ bool warp_runs(uint32_t key, bool act, long long* w, long long off,
                                          bool two_piece, uint32_t& my_cnt) {
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
          const long long u = w[c] - off;
          const unsigned long long s0 = __reduce_add_sync(gm, (unsigned)(u & 0x3ffffff));
          const long long s1 = __reduce_add_sync(gm, (int)(u >> 26));
          w[c] = (long long)s0 + s1 * 67108864ll + (long long)my_cnt * off;
        }
      } else {
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const unsigned long long u = (unsigned long long)(w[c] - off);
          const unsigned long long s0 = __reduce_add_sync(gm, (unsigned)(u & 0x3ffffffu));
          const unsigned long long s1 = __reduce_add_sync(gm, (unsigned)((u >> 26) & 0x3ffffffu));
          const unsigned long long s2 = __reduce_add_sync(gm, (unsigned)(u >> 52));
          w[c] = (long long)(s0 + (s1 << 26) + (s2 << 52)) + (long long)my_cnt * off;
        }
      }
    }
  }
  return act && head;  // only the run's first lane carries the run's sums
}

// Shared-memory atomics on 32-bit shared addresses (no generic-to-shared conversion per use).
// A table entry is EW = 1 + 2D words: [count, lo_0, hi_0, ..., lo_{D-1}, hi_{D-1}] (an odd word
// stride, so random entries spread over the banks); the 64-bit sums are two 32-bit atomics, the
// low word's carry added into the high word.
__device__ __forceinline__ void reds_add(uint32_t a, unsigned v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ void reds_add64(uint32_t a, unsigned long long v) {
  asm volatile(
      "{\n\t.reg .u32 o, t;\n\t"
      "atom.shared.add.u32 o, [%0], %1;\n\t"
      "add.cc.u32 t, o, %1;\n\t"
      "addc.u32 t, %2, 0;\n\t"
      "red.shared.add.u32 [%0+4], t;\n\t}" ::"r"(a),
      "r"((unsigned)v), "r"((unsigned)(v >> 32))
      : "memory");
}

// the (offset) sum of coordinate c held by a table entry
__device__ __forceinline__ unsigned long long bin_entry_sum(const unsigned* ent, int c) {
  return ((unsigned long long)ent[2 + 2 * c] << 32) | ent[1 + 2 * c];
}

// One frame segment [s0, s0 + cnt) of the CTA's range: bin every point into the table (entries
// at shared address ent_s; hash keys at tk).  DENSE: the table is the frame's data box (x reps
// replicas by lane; slots are u16); else the hash table (keys = global cell index; a point
// whose probes fail takes the global atomics).  Coordinates are prefetched two rounds ahead
// (two rounds of 1024 points in flight per SM).
template <int D, typename T, bool FAST, bool DENSE>
__device__ __forceinline__ void bin_segment(const T* __restrict__ pts, int64_t s0, uint32_t cnt,
                                            uint32_t fbase, int64_t fpos0, const GsImg& im,
                                            const BinParams& P, uint32_t ent_s, uint32_t* tk,
                                            uint32_t rep_off, void* __restrict__ slot,
                                            uint32_t* __restrict__ gcnt,
                                            unsigned long long* __restrict__ gqs, int& saw) {
  constexpr int RC = gs_raw_cols<T, D>();
  constexpr int EW = 1 + 2 * D;
  constexpr uint32_t EMPTY = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31;
  const T* __restrict__ src = pts + s0 * RC;
  uint16_t* __restrict__ slot16 = (uint16_t*)slot + s0;
  uint32_t* __restrict__ slot32 = (uint32_t*)slot + s0;
  const uint32_t B = blockDim.x;
  constexpr bool XP = FAST && DENSE;  // the X path (dense tables; the hash path keeps q)
  const long long off = (!XP && (FAST || P.magic_ok)) ? P.Mbits : 0ll;
  T xa[RC], xb[RC];
  {
    const uint32_t i = threadIdx.x;
    const T* pa = src + (size_t)i * RC;
    const T* pb = src + (size_t)(i + B) * RC;
#pragma unroll
    for (int c = 0; c < RC; ++c) {
      xa[c] = i < cnt ? pa[c] : T(0);
      xb[c] = i + B < cnt ? pb[c] : T(0);
    }
  }
  auto point = [&](const T* xc, uint32_t i) {
    uint32_t loc, dloc;
    long long w[D];
    const int st = bin_point<D, T, FAST, XP>(xc, (sizeof(T) == 1 && D > 3) ? fpos0 + i : 0, im, P,
                                         loc, dloc, w);
    uint32_t key = EMPTY;
    if (i < cnt) {
      if (st == 0) {
        if (DENSE || P.s16) slot16[i] = (uint16_t)loc;
        else slot32[i] = fbase + loc;
        key = DENSE ? dloc : fbase + loc;
      } else {
        saw |= st;
      }
    }
    uint32_t my_cnt;
    const bool act = warp_runs<D>(key, key != EMPTY, w, off, XP || P.two_piece, my_cnt);
    if constexpr (DENSE) {
      if (act) {
        const uint32_t a = ent_s + (rep_off + key) * (4 * EW);
        reds_add(a, my_cnt);
#pragma unroll
        for (int c = 0; c < D; ++c) reds_add64(a + 4 + 8 * c, (unsigned long long)w[c]);
      }
    } else {
      const unsigned am = __ballot_sync(kFull, act);
      if (act) {
        // predicated probe loop, then the active lanes reconverge before the atomics (an
        // early-exit loop let the compiler replay the atomic sequence once per exit group)
        const int rl = P.rep_log2;
        const uint32_t tkey = (key << rl) | (lane & ((1u << rl) - 1u));
        uint32_t hsh = __umulhi(tkey * 2654435761u, (unsigned)P.TBL);
        int hit = -1;
#pragma unroll
        for (int probe = 0; probe < kBinProbes; ++probe) {
          if (hit < 0) {
            uint32_t k = tk[hsh];
            if (k == EMPTY) k = atomicCAS(&tk[hsh], EMPTY, tkey);
            if (k == EMPTY || k == tkey) hit = (int)hsh;
            hsh = (hsh + 1 == (unsigned)P.TBL) ? 0u : hsh + 1;
          }
        }
        __syncwarp(am);
        if (hit >= 0) {
          const uint32_t a = ent_s + (uint32_t)hit * (4 * EW);
          reds_add(a, my_cnt);
#pragma unroll
          for (int c = 0; c < D; ++c) reds_add64(a + 4 + 8 * c, (unsigned long long)w[c]);
        } else {
          atomicAdd(&gcnt[key], my_cnt);
#pragma unroll
          for (int c = 0; c < D; ++c)
            atomicAdd(&gqs[(size_t)key * D + c],
                      (unsigned long long)(w[c] - (long long)my_cnt * off));
        }
      }
    }
  };
  auto load = [&](T* x, uint32_t i) {
    const T* pp = src + (size_t)i * RC;
#pragma unroll
    for (int c = 0; c < RC; ++c) x[c] = i < cnt ? pp[c] : T(0);
  };
  // two rounds per trip (the prefetch registers swap roles instead of being copied); every
  // lane runs both halves, so the warp aggregation always sees the whole warp
  for (uint32_t i0 = 0; i0 < cnt; i0 += 2 * B) {
    const uint32_t i = i0 + threadIdx.x;
    T xc[RC];
#pragma unroll
    for (int c = 0; c < RC; ++c) xc[c] = xa[c];
    load(xa, i + 2 * B);
    point(xc, i);
#pragma unroll
    for (int c = 0; c < RC; ++c) xc[c] = xb[c];
    load(xb, i + 3 * B);
    point(xc, i + B);
  }
}

template <int D, typename T, bool FAST, bool DENSE>
__device__ __forceinline__ void bin_range(const T* __restrict__ pts, int64_t p0, int64_t p1,
                                          const GsImg& im, const BinParams& P, unsigned* ent,
                                          uint32_t* tk, void* __restrict__ slot,
                                          uint32_t* __restrict__ gcnt,
                                          unsigned long long* __restrict__ gqs, int& saw) {
  constexpr int EW = 1 + 2 * D;
  const unsigned lane = threadIdx.x & 31;
  const uint32_t vd = P.vd;
  const int reps = P.reps;
  const uint32_t rep_off = DENSE ? (lane % (unsigned)reps) * vd : 0u;
  const uint32_t ent_s = (uint32_t)__cvta_generic_to_shared(ent);
  constexpr bool XP = FAST && DENSE;
  const unsigned long long off = (!XP && (FAST || P.magic_ok)) ? (unsigned long long)P.Mbits : 0ull;
  // segments: one frame each (the dense table holds one frame; a segment's frame base is one
  // constant), also cut every 2^28 points (32-bit offsets inside a segment)
  int64_t s0 = p0;
  int64_t fr = p0 / P.n;
  while (s0 < p1) {
    const int64_t s1 = min(min(p1, (int64_t)((fr + 1) * P.n)), s0 + (int64_t(1) << 28));
    const uint32_t fbase = (uint32_t)(fr * P.vol_frame);
    bin_segment<D, T, FAST, DENSE>(pts, s0, (uint32_t)(s1 - s0), fbase, s0 - fr * P.n, im, P,
                                   ent_s, tk, rep_off, slot, gcnt, gqs, saw);
    __syncthreads();
    if (DENSE) {  // flush this frame's table (replicas summed) and leave it zeroed
      for (uint32_t j = threadIdx.x; j < vd; j += blockDim.x) {
        unsigned cn = 0;
        for (int r = 0; r < reps; ++r) cn += ent[(size_t)(r * vd + j) * EW];
        if (!cn) continue;
        uint32_t L = fbase, rem = j;
        int kk[D];
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const uint32_t dr = rem / P.dstrd[c];
          rem -= dr * P.dstrd[c];
          L += (dr + GS_APRON) * P.strd[c];
          kk[c] = (int)dr + GS_APRON + P.kmin32[c];
        }
        atomicAdd(&gcnt[L], cn);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          // sum(w) - count * off (X path: sum(X) - count * Cr)
          unsigned long long sq = 0ull - (unsigned long long)cn *
                                             (XP ? (unsigned long long)bin_cr(kk[c], P) : off);
          for (int r = 0; r < reps; ++r) sq += bin_entry_sum(ent + (size_t)(r * vd + j) * EW, c);
          atomicAdd(&gqs[(size_t)L * D + c], sq);
        }
        for (int r = 0; r < reps; ++r)
#pragma unroll
          for (int k = 0; k < EW; ++k) ent[(size_t)(r * vd + j) * EW + k] = 0u;
      }
      __syncthreads();
    }
    s0 = s1;
    if (s0 == (fr + 1) * P.n) ++fr;
  }
}

template <int D, typename T>
__global__ void __launch_bounds__(kBinThreads, kBinCtas)
    k_bin(const T* __restrict__ pts, int64_t ntot, const __grid_constant__ BinParams P,
          uint32_t* __restrict__ cnt, unsigned long long* __restrict__ qs, void* __restrict__ slot,
          int* err, int img_w, GsBox* __restrict__ pbox_out = nullptr,
          unsigned* __restrict__ epoch = nullptr, const __grid_constant__ GsBox pbox = GsBox{}) {
  // the predicted box (no bounds pass) becomes the device box here, for K3 (one launch less)
  if (pbox_out && blockIdx.x == 0 && threadIdx.x == 0) {
    *pbox_out = pbox;
    *epoch += 1u;
  }
  constexpr uint32_t EMPTY = 0xffffffffu;
  constexpr int EW = 1 + 2 * D;
  // CTA ranges start on multiples of 4 points (16-byte aligned rows of fp32 d = 3 features)
  const int64_t per = ((ntot + gridDim.x - 1) / gridDim.x + 3) & ~int64_t(3);
  const int64_t p0 = min(ntot, (int64_t)blockIdx.x * per);
  const int64_t p1 = min(ntot, p0 + per);
  __shared__ int s_err;
  if (threadIdx.x == 0) s_err = *err;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* ent = (unsigned*)smem;
  uint32_t* tk = ent + (size_t)EW * P.TBL;
  for (int j = threadIdx.x; j < EW * P.TBL; j += blockDim.x) ent[j] = 0u;
  if (!P.dense)
    for (int j = threadIdx.x; j < P.TBL; j += blockDim.x) tk[j] = EMPTY;
  __syncthreads();
  if (s_err & GS_ERR_SKIP) return;  // non-finite input / box beyond the grid: nothing to bin
  const GsImg im = gs_img(img_w, P.n);
  int saw = 0;
  bool done = false;
  if constexpr (sizeof(T) == 4) {
    if (P.f32fast) {
      if (!P.dense) {
        bin_range<D, T, true, false>(pts, p0, p1, im, P, ent, tk, slot, cnt, qs, saw);
        done = true;
      } else if (P.xpath) {  // dense tables take the fast keys only with the X path
        bin_range<D, T, true, true>(pts, p0, p1, im, P, ent, tk, slot, cnt, qs, saw);
        done = true;
      }
    }
  }
  if (!done) {
    if (P.dense)
      bin_range<D, T, false, true>(pts, p0, p1, im, P, ent, tk, slot, cnt, qs, saw);
    else
      bin_range<D, T, false, false>(pts, p0, p1, im, P, ent, tk, slot, cnt, qs, saw);
  }
  if (saw & 2) atomicOr(err, 1);
  if (saw & 1) atomicOr(err, P.predicted ? 128 : 2);
  if (!P.dense) {
    const unsigned long long off = P.magic_ok ? (unsigned long long)P.Mbits : 0ull;
    for (int j = threadIdx.x; j < P.TBL; j += blockDim.x) {
      const uint32_t key = tk[j];
      if (key == EMPTY) continue;
      const int64_t L = key >> P.rep_log2;
      const unsigned* e = ent + (size_t)j * EW;
      atomicAdd(&cnt[L], e[0]);
#pragma unroll
      for (int c = 0; c < D; ++c)
        atomicAdd(&qs[L * D + c], bin_entry_sum(e, c) - (unsigned long long)e[0] * off);
    }
  }
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
                       double* __restrict__ oS, const int32_t* __restrict__ mnew_dev = nullptr) {
  if (mnew_dev) mnew = *mnew_dev;  // the new cell count straight from the scan (no host read)
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

__global__ void k_idx_set(int m, const uint32_t* __restrict__ key, int32_t* __restrict__ idx,
                          const int32_t* __restrict__ m_dev = nullptr) {
  if (m_dev) m = *m_dev;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) idx[key[i]] = i;
}

// has_converged per frame: fadj[f] = 1 if some cell of f has another
// active cell in its 1-neighbourhood.  D <= 6: batched probes from a shared offset table.
template <int D>
__global__ void k_adjacent(int m, GsBox b, int K, const uint32_t* __restrict__ key,
                           const int32_t* __restrict__ idx, const int32_t* __restrict__ fdone,
                           int32_t* __restrict__ fadj, const int32_t* __restrict__ m_dev = nullptr) {
  if (m_dev) m = *m_dev;
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
// WIDE picks the tuned path (false: u16 frame-local slots of image frames; true: u32 global
// slots of clouds); either instantiation is correct for either slot width (scalar fallback).
template <bool WIDE>
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
  // written straight into pinned host memory over PCIe).  r2: four such groups per lane in
  // flight (their slot loads issued before any gather): one load per lane left the kernel
  // latency-bound (long_scoreboard 95 % of the stalls, 4.5 TB/s)
  const bool vec = s16 && (n % 4) == 0 && (((uintptr_t)slot | (uintptr_t)labels) & 15) == 0;
  const bool vec32 = !s16 && (n % 4) == 0 && (((uintptr_t)slot | (uintptr_t)labels) & 15) == 0;
  for (int64_t f = blockIdx.y; f < nf; f += gridDim.y) {
    const int64_t p0 = f * n;
    const uint32_t fbase = (uint32_t)(f * vf);
    if (!WIDE && vec) {
      const uint2* s4 = reinterpret_cast<const uint2*>((const uint16_t*)slot + p0);
      int4* o4 = reinterpret_cast<int4*>(labels + p0);
      const int64_t n4 = n / 4;
      auto put = [&](int64_t i, const uint2& w) {
        o4[i] = make_int4(__ldg(&lab[fbase + (w.x & 0xffffu)]), __ldg(&lab[fbase + (w.x >> 16)]),
                          __ldg(&lab[fbase + (w.y & 0xffffu)]), __ldg(&lab[fbase + (w.y >> 16)]));
      };
      int64_t i = tid;
      for (; i + 3 * nth < n4; i += 4 * nth) {
        const uint2 w0 = __ldcs(&s4[i]), w1 = __ldcs(&s4[i + nth]), w2 = __ldcs(&s4[i + 2 * nth]),
                    w3 = __ldcs(&s4[i + 3 * nth]);
        put(i, w0);
        put(i + nth, w1);
        put(i + 2 * nth, w2);
        put(i + 3 * nth, w3);
      }
      for (; i < n4; i += nth) put(i, __ldcs(&s4[i]));
    } else if (WIDE && vec32) {
      // u32 slots (global cell indices: clouds): the same shape -- 16-byte slot loads, four
      // groups in flight, 16-byte label stores (one scalar chain per lane ran at 1.7 TB/s)
      const uint4* s4 = reinterpret_cast<const uint4*>((const uint32_t*)slot + p0);
      int4* o4 = reinterpret_cast<int4*>(labels + p0);
      const int64_t n4 = n / 4;
      auto put = [&](int64_t i, const uint4& w) {
        o4[i] = make_int4(__ldg(&lab[w.x]), __ldg(&lab[w.y]), __ldg(&lab[w.z]), __ldg(&lab[w.w]));
      };
      int64_t i = tid;
      for (; i + 3 * nth < n4; i += 4 * nth) {
        const uint4 w0 = __ldcs(&s4[i]), w1 = __ldcs(&s4[i + nth]), w2 = __ldcs(&s4[i + 2 * nth]),
                    w3 = __ldcs(&s4[i + 3 * nth]);
        put(i, w0);
        put(i + nth, w1);
        put(i + 2 * nth, w2);
        put(i + 3 * nth, w3);
      }
      for (; i < n4; i += nth) put(i, __ldcs(&s4[i]));
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
