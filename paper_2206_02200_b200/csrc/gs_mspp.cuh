// gs_mspp.cuh — MS++ baseline: per-point grid mean shift with parallel
// (Jacobi) updates, the comparator of the reference's speed claims.
//
// Reference: module `baselines`, mspp_run (ledger :242-246);
// pins M1-M5 in oracle/gs_oracle.cpp (gso_mspp).  Pipeline on one dataset:
//   K1-K3 (the engine's n-scale phase)  the first grid over the points: lex-sorted cells with
//                                       fixed-point centroids (M1), slot[p], dense index
//   k_mspp_jacobi   (all SMs)           iteration 0's update (M2), a thread per cell
//   k_mspp_disp0    (all SMs)           iteration 0's displacement over the points (M3)
//   k_mspp_loop     (one CTA)           every later iteration with the particles (the previous
//                                       iteration's cells, M4) in shared memory: re-grid
//                                       (bitonic sort by dense key, fixed-point sums), update,
//                                       displacement; then the final cells (M5), the label
//                                       table and the centroids
//   K7 k_label                          labels[p] = lab[slot[p]]
// A first grid larger than one CTA's shared memory (r2: cfg3, cfg5) runs the later iterations
// on all SMs instead, host-driven, one round trip per iteration:
//   k_mspp_bin_g    particles -> the dense grid (count and count * q fixed-point sums, integer
//                   atomics: any order gives the same bits, pin M1/M4)
//   k_occ           the engine's compaction: lex-sorted cells, centroids, idx
//   k_mspp_jacobi_g Eq. (6) per cell (pin M2, as k_mspp_jacobi)
//   k_mspp_disp_g   displacement of every particle (pin M3) and the particle -> cell map of
//                   the initial cells' roots (M4)
//   k_mspp_next_g   the cells become the particles; the grid index is released
// Every fp64 step is the oracle's expression with _rn intrinsics: bit-identical labels,
// centroids, iteration counts and displacements.
#pragma once

#include "gs_common.cuh"

namespace gs {

// Eq. (6) for one cell from the previous state (pin M2): lex-ordered neighbour terms.
template <int D, typename IdxF, typename CntF, typename SF>
__device__ __forceinline__ void mspp_update_cell(const GsBox& b, int64_t L, int i, IdxF idx_at,
                                                 CntF cnt_at, SF s_at, double* out) {
  double num[D];
#pragma unroll
  for (int c = 0; c < D; ++c) num[c] = 0.0;
  uint64_t den = 0;
  int act = 0;
  GsNbrOdometer od;  // the 3^D offsets in lexicographic v order
  od.init(b);
  int K = 1;
#pragma unroll
  for (int c = 0; c < D; ++c) K *= 3;
  for (int t = 0; t < K; ++t) {
    const int j = idx_at(L + od.off);
    od.next(b);
    if (j < 0) continue;
    ++act;
    const uint32_t cj = cnt_at(j);
    den += cj;
#pragma unroll
    for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], __dmul_rn((double)cj, s_at(j, c)));
  }
#pragma unroll
  for (int c = 0; c < D; ++c) out[c] = act <= 1 ? s_at(i, c) : __ddiv_rn(num[c], (double)den);
}

template <int D>
__global__ void k_mspp_jacobi(int m, const GsBox* __restrict__ pb, const uint32_t* __restrict__ ckey,
                              const uint32_t* __restrict__ ccnt, const double* __restrict__ S,
                              const int32_t* __restrict__ idx, double* __restrict__ Snew) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const GsBox b = *pb;
  double o[D];
  mspp_update_cell<D>(
      b, (int64_t)ckey[i], i, [&](int64_t L) { return idx[L]; },
      [&](int j) { return ccnt[j]; }, [&](int j, int c) { return S[(int64_t)j * D + c]; }, o);
#pragma unroll
  for (int c = 0; c < D; ++c) Snew[(int64_t)i * D + c] = o[c];
}

// max over points of |S'(cell of p) - x_p| (pin M3), as the bits of a non-negative double
template <int D, typename T>
__global__ void __launch_bounds__(256) k_mspp_disp0(int64_t n, const T* __restrict__ pts,
                                                     const void* __restrict__ slot,
                                                     const GsBox* __restrict__ pb,
                                                     const int32_t* __restrict__ idx,
                                                     const double* __restrict__ Snew,
                                                     unsigned long long* __restrict__ dmax) {
  unsigned long long best = 0ull;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int r = idx[gs_slot_cell(slot, pb->vol_frame <= 65536, p, 0u)];
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double t = __dsub_rn(Snew[(int64_t)r * D + c], (double)pts[p * D + c]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    best = max(best, (unsigned long long)__double_as_longlong(__dsqrt_rn(acc)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(dmax, best);
}

struct MsppArgs {
  int m0, MS, F, max_iter, vol_small;
  double tol, inv_scale, scale;
  const GsBox* pb;
  const uint32_t* ckey0;   // initial cells: dense keys, counts
  const uint32_t* ccnt0;
  const double* Snew0;     // iteration 0's update of the initial cells
  int32_t* idx;            // the dense grid index (clean -1 outside a run): used when the
                           // frame box does not fit the shared-memory index
  int32_t* lab;            // label table: lab[initial cell key] = final id
  const unsigned long long* disp0;
  double* cent_out;        // final centroids (k x D)
  int* out;                // [k, iterations, converged, error]
  double* disp_hist;       // per-iteration displacement (max_iter)
};

template <int D>
__host__ __device__ constexpr int mspp_bytes_per_slot() {
  // particles: pos D, count, sort key, cell-of | cells: S D, S' D (aliased by the qsums),
  // count, key | root
  return 8 * D + 4 + 8 + 4 + 8 * D + 8 * D + 4 + 4 + 4;
}

template <int D>
__global__ void __launch_bounds__(512, 1) k_mspp_loop(MsppArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ GsBox b;
  __shared__ int s_m, s_mp;
  __shared__ unsigned long long s_disp;
  const int tid = threadIdx.x, T = blockDim.x;
  if (tid == 0) b = *a.pb;
  __syncthreads();
  const int MS = a.MS;
  unsigned char* p = smem;
  double* pos = (double*)p;          p += 8 * (size_t)MS * D;
  double* S = (double*)p;            p += 8 * (size_t)MS * D;
  double* Sn = (double*)p;           p += 8 * (size_t)MS * D;
  long long* qs = (long long*)Sn;    // the re-grid's integer sums die before the update writes S
  uint64_t* sk = (uint64_t*)p;       p += 8 * (size_t)MS;
  uint32_t* pc = (uint32_t*)p;       p += 4 * (size_t)MS;
  int* cof = (int*)p;                p += 4 * (size_t)MS;
  uint32_t* cc = (uint32_t*)p;       p += 4 * (size_t)MS;
  uint32_t* ck = (uint32_t*)p;       p += 4 * (size_t)MS;
  int* root = (int*)p;               p += 4 * (size_t)MS;
  int16_t* sidx = (int16_t*)p;       // vol_small: the frame's dense index in shared memory
  const bool small = a.vol_small != 0;
  auto idx_get = [&](int64_t L) -> int { return small ? (int)sidx[L] : a.idx[L]; };
  auto idx_put = [&](int64_t L, int v) {
    if (small) sidx[L] = (int16_t)v;
    else a.idx[L] = v;
  };
  // particles = the initial cells at their updated positions; the first grid's index entries
  // (written by K3) are released: the clean-grid invariant
  const int m0 = a.m0;
  for (int i = tid; i < m0; i += T) {
    for (int c = 0; c < D; ++c) pos[i * D + c] = a.Snew0[(int64_t)i * D + c];
    pc[i] = a.ccnt0[i];
    root[i] = i;
    a.idx[a.ckey0[i]] = -1;
  }
  if (small)
    for (int j = tid; j < (int)b.vol_frame; j += T) sidx[j] = -1;
  if (tid == 0) {
    s_mp = m0;
    s_disp = *a.disp0;
  }
  __syncthreads();
  int it = 1;
  const double d0 = __longlong_as_double((long long)s_disp);
  if (tid == 0 && a.disp_hist) a.disp_hist[0] = d0;
  bool conv = d0 < a.tol;
  bool final_pass = conv || it >= a.max_iter;
  for (;;) {
    // ---- re-grid the particles (pins M1, M4): sort by dense key, segments, fixed-point sums
    const int mp = s_mp;
    int P = 1;
    while (P < mp) P <<= 1;
    for (int i = tid; i < P; i += T) {
      if (i < mp) {
        int64_t L = 0;
        for (int c = 0; c < D; ++c) {
          const int64_t k = gs_grid_coord(pos[i * D + c], b.h, b.inv_h);
          L += (k - b.kmin[c]) * b.stride[c];
        }
        sk[i] = ((uint64_t)(uint32_t)L << 32) | (uint32_t)i;
      } else {
        sk[i] = ~0ull;
      }
    }
    __syncthreads();
    for (int k2 = 2; k2 <= P; k2 <<= 1) {
      for (int j = k2 >> 1; j > 0; j >>= 1) {
        for (int i = tid; i < P; i += T) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const uint64_t x = sk[i], y = sk[ixj];
            if ((x > y) == ((i & k2) == 0)) {
              sk[i] = y;
              sk[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    // segment heads -> cell ranks (serial prefix by one warp: m <= MS is small)
    if (tid < 32) {
      int run = 0;
      for (int base = 0; base < mp; base += 32) {
        const int j = base + tid;
        const bool head = j < mp && (j == 0 || (sk[j] >> 32) != (sk[j - 1] >> 32));
        const unsigned bm = __ballot_sync(0xffffffffu, head);
        const int g = run + __popc(bm & ((1u << tid) - 1u)) + (head ? 1 : 0) - 1;
        if (j < mp) cof[(uint32_t)sk[j]] = g;
        if (head) ck[g] = (uint32_t)(sk[j] >> 32);
        run += __popc(bm);
      }
      if (tid == 0) s_m = run;
    }
    __syncthreads();
    const int m = s_m;
    for (int g = tid; g < m; g += T) {
      cc[g] = 0u;
      for (int c = 0; c < D; ++c) qs[g * D + c] = 0;
    }
    __syncthreads();
    for (int i = tid; i < mp; i += T) {  // integer sums: any order gives the same bits
      const int g = cof[i];
      atomicAdd(&cc[g], pc[i]);
      const int64_t L = ck[g];
      for (int c = 0; c < D; ++c) {
        const int64_t kc = (L / b.stride[c]) % b.ext[c] + b.kmin[c];
        const long long q = gs_fixq(pos[i * D + c], kc, b.h, a.scale);
        atomicAdd((unsigned long long*)&qs[g * D + c], (unsigned long long)((long long)pc[i] * q));
      }
    }
    __syncthreads();
    for (int g = tid; g < m; g += T) {
      const int64_t L = ck[g];
      for (int c = 0; c < D; ++c) {
        const int64_t kc = (L / b.stride[c]) % b.ext[c] + b.kmin[c];
        S[g * D + c] = gs_fix_centroid(kc, qs[g * D + c], cc[g], b.h, a.inv_scale);
      }
    }
    __syncthreads();
    if (final_pass) {  // pin M5: the final cells; ids = lex ranks
      for (int g = tid; g < m; g += T)
        for (int c = 0; c < D; ++c) a.cent_out[(int64_t)g * D + c] = S[g * D + c];
      for (int c0 = tid; c0 < m0; c0 += T) a.lab[a.ckey0[c0]] = cof[root[c0]];
      if (tid == 0) {
        a.out[0] = m;
        a.out[1] = it;
        a.out[2] = conv ? 1 : 0;
      }
      return;
    }
    // ---- update (pin M2) with the cells' dense index
    for (int g = tid; g < m; g += T) idx_put(ck[g], g);
    if (tid == 0) s_disp = 0ull;
    __syncthreads();
    for (int g = tid; g < m; g += T) {
      double o[D];
      mspp_update_cell<D>(
          b, (int64_t)ck[g], g, idx_get, [&](int j) { return cc[j]; },
          [&](int j, int c) { return S[j * D + c]; }, o);
      for (int c = 0; c < D; ++c) Sn[g * D + c] = o[c];
    }
    __syncthreads();
    for (int g = tid; g < m; g += T) idx_put(ck[g], -1);
    // ---- displacement of every particle (pin M3); particles -> their cells (M4)
    unsigned long long best = 0ull;
    for (int i = tid; i < mp; i += T) {
      const int g = cof[i];
      double acc = 0.0;
      for (int c = 0; c < D; ++c) {
        const double t = __dsub_rn(Sn[g * D + c], pos[i * D + c]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
      }
      best = max(best, (unsigned long long)__double_as_longlong(__dsqrt_rn(acc)));
    }
    if (best) atomicMax(&s_disp, best);
    for (int c0 = tid; c0 < m0; c0 += T) root[c0] = cof[root[c0]];
    __syncthreads();
    for (int g = tid; g < m; g += T) {
      for (int c = 0; c < D; ++c) pos[g * D + c] = Sn[g * D + c];
      pc[g] = cc[g];
    }
    const double dsp = __longlong_as_double((long long)s_disp);
    if (tid == 0) {
      s_mp = m;
      if (a.disp_hist) a.disp_hist[it] = dsp;
    }
    ++it;
    conv = dsp < a.tol;
    final_pass = conv || it >= a.max_iter;
    __syncthreads();
  }
}

// ---- the all-SM loop (first grids beyond one CTA)
__global__ void k_iota(int m, int32_t* __restrict__ v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) v[i] = i;
}

template <int D>
__global__ void k_mspp_bin_g(int mp, const double* __restrict__ pos,
                             const uint32_t* __restrict__ pc, const GsBox* __restrict__ pb,
                             double scale, uint32_t* __restrict__ cnt,
                             unsigned long long* __restrict__ qs, uint32_t* __restrict__ pkey,
                             unsigned* __restrict__ epoch, unsigned* __restrict__ ticket,
                             int* __restrict__ err) {
  const GsBox b = *pb;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0) {  // a fresh compaction epoch and tile ticket for the k_occ that follows
    *epoch += 1u;
    *ticket = 0u;
  }
  if (i >= mp) return;
  int64_t L = 0, kc[D];
  bool out = false;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    kc[c] = gs_grid_coord(pos[(int64_t)i * D + c], b.h, b.inv_h);
    const int64_t r = kc[c] - b.kmin[c];
    out |= r < 0 || r >= b.ext[c];
    L += r * b.stride[c];
  }
  if (out) {  // (a mean of points of the box stays in it)
    atomicOr(err, 2);
    return;
  }
  pkey[i] = (uint32_t)L;
  atomicAdd(&cnt[L], pc[i]);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const long long q = gs_fixq(pos[(int64_t)i * D + c], kc[c], b.h, scale);
    atomicAdd(&qs[L * D + c], (unsigned long long)((long long)pc[i] * q));
  }
}

template <int D>
__global__ void k_mspp_jacobi_g(const unsigned* __restrict__ m_ptr, const GsBox* __restrict__ pb,
                                const uint32_t* __restrict__ ckey,
                                const uint32_t* __restrict__ ccnt, const double* __restrict__ S,
                                const int32_t* __restrict__ idx, double* __restrict__ Snew) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int)*m_ptr) return;
  const GsBox b = *pb;
  double o[D];
  mspp_update_cell<D>(
      b, (int64_t)ckey[i], i, [&](int64_t L) { return idx[L]; },
      [&](int j) { return ccnt[j]; }, [&](int j, int c) { return S[(int64_t)j * D + c]; }, o);
#pragma unroll
  for (int c = 0; c < D; ++c) Snew[(int64_t)i * D + c] = o[c];
}

template <int D>
__global__ void __launch_bounds__(256) k_mspp_disp_g(int mp, const double* __restrict__ pos,
                                                      const uint32_t* __restrict__ pkey,
                                                      const int32_t* __restrict__ idx,
                                                      const double* __restrict__ Snew,
                                                      unsigned long long* __restrict__ dmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long best = 0ull;
  if (i < mp) {
    const int g = idx[pkey[i]];
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double t = __dsub_rn(Snew[(int64_t)g * D + c], pos[(int64_t)i * D + c]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    best = (unsigned long long)__double_as_longlong(__dsqrt_rn(acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(dmax, best);
}

// root[c0] <- the cell (rank) of the initial cell's particle; final: lab[initial key] = it
__global__ void k_mspp_root_g(int m0, int32_t* __restrict__ root, const uint32_t* __restrict__ pkey,
                              const int32_t* __restrict__ idx, const uint32_t* __restrict__ ckey0,
                              int32_t* __restrict__ lab) {
  const int c0 = blockIdx.x * blockDim.x + threadIdx.x;
  if (c0 >= m0) return;
  const int g = idx[pkey[root[c0]]];
  if (lab) lab[ckey0[c0]] = g;
  else root[c0] = g;
}

// the m cells become the particles (positions Snew, counts); the grid index is released
template <int D>
__global__ void k_mspp_next_g(const unsigned* __restrict__ m_ptr, const double* __restrict__ Snew,
                              const uint32_t* __restrict__ ccnt, const uint32_t* __restrict__ ckey,
                              double* __restrict__ pos, uint32_t* __restrict__ pc,
                              int32_t* __restrict__ idx) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int)*m_ptr) return;
#pragma unroll
  for (int c = 0; c < D; ++c) pos[(int64_t)g * D + c] = Snew[(int64_t)g * D + c];
  pc[g] = ccnt[g];
  idx[ckey[g]] = -1;
}

}  // namespace gs
