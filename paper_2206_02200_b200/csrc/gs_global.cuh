// gs_global.cuh — the sweep of the global path (frames too large for one CTA's smem).
//
// Same design as K8's sweep (gs_resident.cuh), with the cell state in L2-resident global
// memory:
//   k_nbr_count / k_nbr_fill (all SMs)  neighbour census, then per cell {slot, C'} records of
//                                        its lex-earlier active neighbours, the C'*S_old
//                                        products and slots of itself and its lex-later ones,
//                                        ΣC' and RN(1/ΣC')
//   k_sweep_kahn (one CTA)               Kahn frontier over the sweep DAG: each level is
//                                        updated with every operand final (a lane group per
//                                        cell), then releases its lex-later neighbours
// Operands and order of the fp64 adds are exactly the serial sweep's (pins P2/P3).
#pragma once

#include <cooperative_groups.h>

#include <climits>

#include "gs_common.cuh"

namespace gs {

__device__ __forceinline__ double gl_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double fa = fabs(a);
  if (!(fa < 0x1p+1000) || (fa < 0x1p-900 && a != 0.0)) return gs_ddiv_slow(a, b);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}

// Neighbour lists at a fixed stride of KP entries (no census, no scan, no host round trip):
// per cell the Q-row of every active neighbour in lex order (earlier neighbour j -> P1 row
// m+1+j = C'*S_new, itself / later -> row j = C'*S_old), padded with the zero row m; #active,
// #earlier, ΣC' and RN(1/ΣC'); Q row i = C'*S_old (S_old itself when the cell has no active
// neighbour but itself, pin P3).  Frozen frames: nbn = 0, Q row = S_old.
// Lexicographic neighbour offsets (v in {-1,0,1}^D, dim 0 most significant: the odometer's
// order) as linear deltas of the frame box, one per thread of the block (D <= 6: K <= 729).
template <int D>
__device__ __forceinline__ void nbr_offsets_smem(const GsBox& b, int K, int* offs) {
  for (int t = threadIdx.x; t < K; t += blockDim.x) {
    int r = t;
    int64_t off = 0;
    for (int c = D - 1; c >= 0; --c) {
      off += (int64_t)(r % 3 - 1) * b.stride[c];
      r /= 3;
    }
    offs[t] = (int)off;
  }
}

template <int D>
__global__ void k_nbr_lists(int m, GsBox b, int K, int KP, const uint32_t* __restrict__ ckey,
                            const uint32_t* __restrict__ ccnt, const double* __restrict__ S0,
                            const int32_t* __restrict__ idx, const int32_t* __restrict__ fdone,
                            uint32_t* __restrict__ lists, int32_t* __restrict__ nbn,
                            int32_t* __restrict__ nbe, uint32_t* __restrict__ den,
                            double* __restrict__ rden, double* __restrict__ Q,
                            int32_t* __restrict__ fm, int own_lo = 0, int own_hi = INT_MAX,
                            int32_t* __restrict__ npend = nullptr) {
  // probes in batches of 27 from a shared offset table: the loads of a batch are independent
  // (one L2 round trip per batch instead of one per probe behind the odometer and the stores)
  // own_lo/own_hi (multi-GPU slabs, gs_dist): cells outside [own_lo, own_hi) are halo cells
  // of the neighbouring slabs -- frozen here (their rows are written by the caller); npend =
  // the own earlier neighbours, the sweep's pending counts (an own cell does not wait on the
  // lower halo: it is final before this slab's sweep starts)
  constexpr int KMAX = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : D == 5 ? 243 : 729;
  constexpr int B = KMAX < 27 ? KMAX : 27;
  __shared__ int offs[KMAX];
  nbr_offsets_smem<D>(b, KMAX, offs);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0)
    for (int c = 0; c < D; ++c) Q[(int64_t)m * D + c] = 0.0;  // the zero row
  if (i >= m) return;
  const int64_t L = ckey[i];
  const int64_t f = L / b.vol_frame;
  uint32_t* li = lists + (int64_t)i * KP;
  if (fdone[f] || i < own_lo || i >= own_hi) {
    nbn[i] = nbe[i] = 0;
    if (npend) npend[i] = 0;
    den[i] = ccnt[i];
    for (int c = 0; c < D; ++c) Q[(int64_t)i * D + c] = S0[(int64_t)i * D + c];
    return;
  }
  atomicAdd(&fm[f], 1);
  int n = 0, e = 0, eo = 0;
  uint32_t s = 0;
  const uint32_t P1ROW = (uint32_t)m + 1u, ZROW = (uint32_t)m;
  for (int t0 = 0; t0 < KMAX; t0 += B) {
    int jb[B];
#pragma unroll
    for (int u = 0; u < B; ++u) jb[u] = __ldg(&idx[L + offs[t0 + u]]);
    uint32_t cb[B];
#pragma unroll
    for (int u = 0; u < B; ++u) cb[u] = jb[u] >= 0 ? __ldg(&ccnt[jb[u]]) : 0u;
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int32_t j = jb[u];
      if (j < 0) continue;
      s += cb[u];
      li[n++] = j < i ? P1ROW + (uint32_t)j : (uint32_t)j;
      e += j < i;
      eo += j < i && j >= own_lo;
    }
  }
  for (int t = n; t < KP; ++t) li[t] = ZROW;
  nbn[i] = n;
  nbe[i] = e;
  if (npend) npend[i] = eo;
  den[i] = s;
  rden[i] = __drcp_rn((double)s);
  const double ci = (double)ccnt[i];
  for (int c = 0; c < D; ++c)
    Q[(int64_t)i * D + c] =
        n <= 1 ? S0[(int64_t)i * D + c] : __dmul_rn(ci, S0[(int64_t)i * D + c]);
}

// The global path's sweep: ONE CTA runs Kahn frontiers over the whole (multi-frame) cell set
// with the state in L2 (`Q`, lists, per-cell metadata; operands read with ld.global.cg since
// they are written during the kernel).  Per level: every warp updates the frontier's cells,
// one lane per (cell, coordinate) -- the serial sweep's operands in lex order, +0.0 padding --
// then every thread releases the successors of one frontier cell (pending counts packed as
// bytes in shared memory, the queue in shared memory as u16 when the cells fit, else both in
// global scratch).  One block barrier per level.
template <int D>
constexpr int sweep_global_threads() { return D <= 3 ? 1024 : 512; }  // d > 3: 128 registers

template <int D>
__global__ void __launch_bounds__(sweep_global_threads<D>(), 1) k_sweep_global(
    int m, int KP, const uint32_t* __restrict__ lists, const int32_t* __restrict__ nbn,
    const int32_t* __restrict__ nbe, const uint32_t* __restrict__ ccnt,
    const uint32_t* __restrict__ den, const double* __restrict__ rden, double* Q,
    unsigned* pend_g, unsigned* queue_g, int in_smem, long long* prof = nullptr,
    const int32_t* __restrict__ pinit = nullptr) {
  // prof (diagnostics, GS_TRACE_GLOBAL): per level [width, start, per-warp update end x 32,
  // per-warp release end x 32] clock stamps, plain stores (no atomics on the path)
  extern __shared__ __align__(16) unsigned char dsm[];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = T >> 5;
  unsigned* pend = in_smem ? (unsigned*)dsm : pend_g;                  // (m + 3) / 4 words
  uint16_t* q16 = (uint16_t*)(dsm + 4 * (((size_t)m + 3) / 4 + 1));   // m entries (u16)
  __shared__ int tail;
  auto q_get = [&](int k) -> int { return in_smem ? (int)q16[k] : (int)queue_g[k]; };
  auto q_put = [&](int k, int v) {
    if (in_smem)
      q16[k] = (uint16_t)v;
    else
      queue_g[k] = (unsigned)v;
  };
  if (tid == 0) tail = 0;
  for (int w = tid; w < (m + 3) / 4; w += T) pend[w] = 0u;
  __syncthreads();
  for (int i = tid; i < m; i += T) {
    const int e = pinit ? pinit[i] : nbe[i];  // pending predecessors
    if (e > 0) atomicAdd(&pend[i >> 2], (unsigned)e << (8 * (i & 3)));
    else q_put(atomicAdd(&tail, 1), i);
  }
  constexpr int CPW = 32 / D;
  const int q = lane / D, c = lane - (lane / D) * D;
  const uint32_t P1ROW = (uint32_t)m + 1u;
  int qhead = 0, plev = 0;
  for (;;) {
    __syncthreads();  // the previous level's appends are complete
    const int lev_end = *(volatile int*)&tail;
    if (qhead >= lev_end) break;
    long long* pl = (prof && plev < 2000) ? prof + (int64_t)plev * 66 : nullptr;
    if (pl && tid == 0) {
      pl[0] = lev_end - qhead;
      pl[1] = clock64();
    }
    // ---- update the frontier
    for (int base = qhead + warp * CPW; base < lev_end; base += nwarps * CPW) {
      const int k = base + q;
      const bool act = q < CPW && k < lev_end;
      const int i = act ? q_get(k) : 0;
      const int n = act ? nbn[i] : 0;
      if (n > 1) {  // else: frozen or no active neighbour but itself (Q row = S_old, P3)
        const uint4* ls = (const uint4*)(lists + (int64_t)i * KP);
        double num = 0.0;
        if constexpr (D <= 3) {
          // every word and operand up front (L2 latency dominates), then the whole padded
          // chain: the zero-row padding adds +0.0
          constexpr int NW = (D == 1 ? 3 : D == 2 ? 9 : 27) / 4 + 1;
          uint4 r[NW];
#pragma unroll
          for (int w = 0; w < NW; ++w) r[w] = __ldg(&ls[w]);
          double v[NW][4];
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            v[w][0] = __ldcg(&Q[(int64_t)r[w].x * D + c]);
            v[w][1] = __ldcg(&Q[(int64_t)r[w].y * D + c]);
            v[w][2] = __ldcg(&Q[(int64_t)r[w].z * D + c]);
            v[w][3] = __ldcg(&Q[(int64_t)r[w].w * D + c]);
          }
#pragma unroll
          for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int t = 0; t < 4; ++t) num = __dadd_rn(num, v[w][t]);
        } else {
          // blocks of 4 words (16 terms): each block's loads issued together, the next
          // block's in flight while this one is added (L2 latency, not the adds, is the cost)
          const int nq = (n + 3) >> 2;
          constexpr int WB = 4;
          uint4 ra[WB], rb[WB];
          double va[WB][4], vb[WB][4];
          auto fetch = [&](uint4 (&r)[WB], double (&v)[WB][4], int w0) {
#pragma unroll
            for (int w = 0; w < WB; ++w) r[w] = __ldg(&ls[min(w0 + w, KP / 4 - 1)]);
#pragma unroll
            for (int w = 0; w < WB; ++w) {
              const bool in = w0 + w < nq;  // beyond the list: +0.0 terms
              v[w][0] = in ? __ldcg(&Q[(int64_t)r[w].x * D + c]) : 0.0;
              v[w][1] = in ? __ldcg(&Q[(int64_t)r[w].y * D + c]) : 0.0;
              v[w][2] = in ? __ldcg(&Q[(int64_t)r[w].z * D + c]) : 0.0;
              v[w][3] = in ? __ldcg(&Q[(int64_t)r[w].w * D + c]) : 0.0;
            }
          };
          auto fold = [&](const double (&v)[WB][4]) {
#pragma unroll
            for (int w = 0; w < WB; ++w)
#pragma unroll
              for (int t = 0; t < 4; ++t) num = __dadd_rn(num, v[w][t]);
          };
          fetch(ra, va, 0);
          for (int w0 = 0; w0 < nq; w0 += 2 * WB) {
            if (w0 + WB < nq) fetch(rb, vb, w0 + WB);
            fold(va);
            if (w0 + WB >= nq) break;
            if (w0 + 2 * WB < nq) fetch(ra, va, w0 + 2 * WB);
            fold(vb);
          }
        }
        const double s1 = gl_div(num, (double)den[i], rden[i]);
        __stcg(&Q[((int64_t)P1ROW + i) * D + c], __dmul_rn((double)ccnt[i], s1));
        __stcg(&Q[(int64_t)i * D + c], s1);
      }
    }
    if (pl && lane == 0) pl[2 + warp] = clock64();
    // (no barrier here: the release only prepares the NEXT frontier, which starts after the
    // loop-top barrier, by when every row of this one is final)
    // ---- release the frontier's later neighbours: d <= 3 a thread per frontier cell (<= 13
    //      successors), d > 3 a warp per cell with its lanes over the successors (up to 121
    //      for d = 5: a thread per cell would serialise them)
    constexpr int RW = D <= 3 ? 1 : 32;  // lanes per frontier cell
    for (int k = qhead + tid / RW; k < lev_end; k += T / RW) {
      const int i = q_get(k);
      const int n = nbn[i], e = nbe[i];
      const uint32_t* li = lists + (int64_t)i * KP;
      for (int t = e + 1 + (RW == 1 ? 0 : lane); t < n; t += RW) {  // entry e: the cell itself
        const int j = (int)__ldg(&li[t]);
        const unsigned sh = 8 * (j & 3);
        const unsigned old = atomicSub(&pend[j >> 2], 1u << sh);
        if (((old >> sh) & 0xffu) == 1u) q_put(atomicAdd(&tail, 1), j);
      }
    }
    if (pl && lane == 0) pl[34 + warp] = clock64();
    ++plev;
    qhead = lev_end;
  }
  if (prof && tid == 0) prof[2000 * 66] = plev;
}

// census: number of active neighbours and of lex-earlier ones; frozen frames -> 0
__global__ void k_nbr_count(int m, GsBox b, int K, const uint32_t* __restrict__ ckey,
                            const int32_t* __restrict__ idx, const int32_t* __restrict__ fdone,
                            int32_t* __restrict__ nbn, int32_t* __restrict__ nbe,
                            int32_t* __restrict__ ecnt, int32_t* __restrict__ lcnt,
                            int32_t* __restrict__ fm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int64_t L = ckey[i];
  const int64_t f = L / b.vol_frame;
  if (fdone[f]) {
    nbn[i] = nbe[i] = ecnt[i] = lcnt[i] = 0;
    return;
  }
  atomicAdd(&fm[f], 1);
  GsNbrOdometer od;
  od.init(b);
  int n = 0, e = 0;
  for (int t = 0; t < K; ++t) {
    const int32_t j = __ldg(&idx[L + od.off]);
    n += (j >= 0);
    e += (j >= 0) & (j < i);
    od.next(b);
  }
  nbn[i] = n;
  nbe[i] = e;
  ecnt[i] = e;
  lcnt[i] = n - e;
}

// records at the scanned offsets
__global__ void k_nbr_fill(int m, GsBox b, int K, const uint32_t* __restrict__ ckey,
                           const uint32_t* __restrict__ ccnt, const double* __restrict__ S0,
                           const int32_t* __restrict__ idx, const int32_t* __restrict__ nbn,
                           const int32_t* __restrict__ eoff, const int32_t* __restrict__ loff,
                           unsigned long long* __restrict__ erec, double* __restrict__ lprod,
                           int32_t* __restrict__ lsucc, uint32_t* __restrict__ den,
                           double* __restrict__ rden) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int d = b.d;
  if (nbn[i] == 0) {  // frozen frame
    den[i] = ccnt[i];
    return;
  }
  const int64_t L = ckey[i];
  GsNbrOdometer od;
  od.init(b);
  int ne = 0, nl = 0;
  uint32_t s = 0;
  const int e0 = eoff[i], l0 = loff[i];
  for (int t = 0; t < K; ++t) {
    const int32_t j = __ldg(&idx[L + od.off]);
    od.next(b);
    if (j < 0) continue;
    const uint32_t w = ccnt[j];
    s += w;
    if (j < i) {
      erec[e0 + ne++] = ((unsigned long long)w << 32) | (uint32_t)j;
    } else {
      lsucc[l0 + nl] = j;
      double* dst = lprod + (int64_t)(l0 + nl++) * d;
      for (int c = 0; c < d; ++c) dst[c] = __dmul_rn((double)w, S0[(int64_t)j * d + c]);
    }
  }
  den[i] = s;
  rden[i] = __drcp_rn((double)s);
}


// Lanes per cell in the cooperative update.
template <int D>
__host__ __device__ constexpr int sweep_group() {
  return 32;  // one warp per cell: no intra-warp serialisation between cells
}

// One CTA.  pend/queue live in dynamic shared memory when 8*m bytes fit (smem_cells >= m),
// else in the global scratch arrays.  Dynamic smem layout: [stage: blockDim*D doubles]
// [pend: smem_cells ints][queue: smem_cells ints].
template <int D>
__global__ void __launch_bounds__(1024, 1) k_sweep_kahn(
    int m, int smem_cells, const int32_t* __restrict__ nbn, const int32_t* __restrict__ nbe,
    const int32_t* __restrict__ eoff, const int32_t* __restrict__ loff,
    const unsigned long long* __restrict__ erec, const double* __restrict__ lprod,
    const int32_t* __restrict__ lsucc, const uint32_t* __restrict__ den,
    const double* __restrict__ rden, const double* __restrict__ S0, double* S1, int* pend_g,
    int* queue_g, long long* dbg) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int tid = threadIdx.x, T = blockDim.x;
  constexpr int G = sweep_group<D>();
  double* stage = (double*)dsm;
  int* sq = (int*)(stage + (size_t)T * D);
  const bool in_smem = m <= smem_cells;
  int* pend = in_smem ? sq : pend_g;
  volatile int* queue = in_smem ? sq + smem_cells : queue_g;
  const int grp = tid / G, g = tid % G, ngroups = T / G;
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) & ~(G - 1)));
  double* stg = stage + (size_t)grp * G * D;
  __shared__ unsigned tail;
  if (tid == 0) tail = 0u;
  __syncthreads();
  for (int i = tid; i < m; i += T) {
    pend[i] = nbe[i];
    if (nbe[i] == 0) queue[atomicAdd(&tail, 1u)] = i;
  }
  int qhead = 0;
  for (;;) {
    __syncthreads();  // the previous level's appends are complete
    const int lev_end = (int)*(volatile unsigned*)&tail;
    __syncthreads();  // everyone holds lev_end before new appends
    if (qhead >= lev_end) break;
    if (dbg && tid == 0) {
      atomicAdd((unsigned long long*)&dbg[0], 1ull);
      atomicAdd((unsigned long long*)&dbg[1], (unsigned long long)(lev_end - qhead));
    }
    const long long tl0 = clock64();
    for (int k = qhead + grp; k < lev_end; k += ngroups) {
      const int i = queue[k];
      const int n = nbn[i], e = nbe[i];
      if (n <= 1) {  // isolated or frozen: centroid kept bit-for-bit (pin P3)
        if (g < D) S1[(int64_t)i * D + g] = S0[(int64_t)i * D + g];
      } else {
        double num = 0.0;  // lane g < D accumulates coordinate g
        for (int t0 = 0; t0 < n; t0 += G) {
          const int t = t0 + g;
          if (t < n) {
            if (t < e) {  // earlier neighbour: its NEW centroid
              const unsigned long long r = erec[eoff[i] + t];
              const int64_t j = (uint32_t)r;
              const double w = (double)(uint32_t)(r >> 32);
#pragma unroll
              for (int c = 0; c < D; ++c) stg[g * D + c] = __dmul_rn(w, __ldcg(&S1[j * D + c]));
            } else {  // itself / later neighbour: precomputed C'*S_old
              const double* lp = lprod + (int64_t)(loff[i] + (t - e)) * D;
#pragma unroll
              for (int c = 0; c < D; ++c) stg[g * D + c] = lp[c];
            }
          }
          __syncwarp(gmask);
          if (g < D) {
            const int len = min(G, n - t0);
#pragma unroll 4
            for (int u = 0; u < len; ++u) num = __dadd_rn(num, stg[u * D + g]);
          }
          __syncwarp(gmask);
        }
        if (g < D) S1[(int64_t)i * D + g] = gl_div(num, (double)den[i], rden[i]);
      }
      // release the lex-later neighbours (self is the first late record), in parallel
      const int l0 = loff[i] + 1, ns = n - e - 1;
      for (int t = g; t < ns; t += G) {
        const int j = lsucc[l0 + t];
        if (atomicSub(&pend[j], 1) == 1) queue[atomicAdd(&tail, 1u)] = j;
      }
    }
    if (dbg && tid == 0)
      atomicAdd((unsigned long long*)&dbg[2], (unsigned long long)(clock64() - tl0));
    qhead = lev_end;
  }
}

// ---------------------------------------------------------------- cluster sweep
// The same Kahn-frontier sweep spread over a thread-block cluster of NC CTAs (one per SM):
// the single-CTA sweep above is bound by one SM's bandwidth to L2 (every term of a cell is a
// scattered 8-byte row read: cfg5's 316-cell frontiers took ~14 K cycles per level to update,
// cfg3's d = 5 lists ~18 K).  Cell j is owned by CTA j % NC, which keeps j's pending count and
// its frontier queue in its shared memory; a CTA updates the frontier cells it owns (operand
// rows and lists in L2, exactly the single-CTA update) and releases their successors with
// atomics on the OWNER's shared memory (DSMEM); a cluster barrier separates levels (its
// release/acquire orders the row stores and the queue appends).  Termination: every CTA adds
// the number of cells it updated to a per-level counter in CTA 0 (three buffers, so a counter
// is read by everyone before it is reused), and all CTAs stop when the running total reaches m.
// Operands and add order are the serial sweep's: bit-identical results.
template <int D>
constexpr int sweep_cluster_threads() { return 512; }  // 128 registers: no spills at d = 3

// dynamic shared memory of the cluster sweep: pending counts + two queues per owned cell,
// and for d > 3 a 128-entry staging tile of operand rows per warp
template <int D>
__host__ __device__ constexpr size_t sweep_cluster_smem(int mloc) {
  return (((size_t)12 * mloc + 15) & ~(size_t)15) +
         (D > 3 ? (size_t)(sweep_cluster_threads<D>() / 32) * 128 * D * 8 : 0);
}

template <int D>
__global__ void __launch_bounds__(sweep_cluster_threads<D>(), 1) k_sweep_cluster(
    int m, int KP, const uint32_t* __restrict__ lists, const int32_t* __restrict__ nbn,
    const int32_t* __restrict__ nbe, const uint32_t* __restrict__ ccnt,
    const uint32_t* __restrict__ den, const double* __restrict__ rden, double* Q,
    long long* prof = nullptr, const int32_t* __restrict__ pinit = nullptr) {
  // prof (diagnostics, GS_TRACE_GLOBAL): per level and CTA [width, start, update end,
  // release end, barrier end] clock stamps (an extra block barrier after the update)
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int NC = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char dsm[];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = T >> 5;
  const int mloc = (m + NC - 1) / NC;          // cells owned by this CTA: j = rank + NC*t
  unsigned* pend = (unsigned*)dsm;              // mloc pending counts
  // two frontier buffers by level parity: level L reads qbuf[L & 1] (filled during level L-1)
  // while its releases append to qbuf[(L + 1) & 1], so a CTA's level boundary never moves
  // under it; the buffer is emptied by its owner after its last read, before the barrier
  unsigned* qbuf0 = pend + mloc;
  unsigned* qbuf1 = pend + 2 * mloc;
  const size_t stage_off = ((size_t)12 * mloc + 15) & ~(size_t)15;  // d > 3: per-warp tiles
  __shared__ unsigned tails[2];
  __shared__ unsigned done_cnt[3];
  if (tid == 0) {
    tails[0] = tails[1] = 0;
    done_cnt[0] = done_cnt[1] = done_cnt[2] = 0;
  }
  __syncthreads();
  for (int t = tid; t < mloc; t += T) {
    const int i = rank + NC * t;
    if (i >= m) break;
    const int e = pinit ? pinit[i] : nbe[i];  // pending predecessors
    pend[t] = (unsigned)e;
    if (e == 0) qbuf0[atomicAdd(&tails[0], 1u)] = (unsigned)i;
  }
  unsigned* cnt0 = cluster.map_shared_rank(&done_cnt[0], 0);
  constexpr int CPW = 32 / D;
  const int q = lane / D, c = lane - (lane / D) * D;
  const uint32_t P1ROW = (uint32_t)m + 1u;
  int level = 0;
  long long total = 0;
  cluster.sync();  // every CTA's pending counts and initial queue are in place
  for (;;) {
    const int cur = level & 1;
    unsigned* queue = cur ? qbuf1 : qbuf0;
    const int lev_end = (int)*(volatile unsigned*)&tails[cur];
    const int qhead = 0;
    long long* pl = (prof && level < 1000) ? prof + ((int64_t)level * 16 + rank) * 5 : nullptr;
    if (pl && tid == 0) {
      pl[0] = lev_end;
      pl[1] = clock64();
    }
    const int nxt = cur ^ 1;
    auto release_one = [&](int j) {  // successor j: its owner's pending count, next queue
      const int own = j % NC;
      unsigned* pj = cluster.map_shared_rank(pend + j / NC, own);
      if (atomicSub(pj, 1u) == 1u) {
        unsigned* tl = cluster.map_shared_rank(&tails[nxt], own);
        unsigned* qd = cluster.map_shared_rank(nxt ? qbuf1 : qbuf0, own);
        qd[atomicAdd(tl, 1u)] = (unsigned)j;
      }
    };
    if constexpr (D > 3) {
      // ---- d > 3: a warp per frontier cell.  Lane l loads list word l of each 128-entry
      // chunk (one L2 round trip for the whole chunk instead of one per 16 entries), releases
      // the successors among its 4 entries right away (they are processed after the level's
      // cluster barrier, by when this cell's row is stored), loads the 4 entries' operand rows
      // into a per-warp staging tile, and lane c < D then adds the chunk's terms in list order.
      double* stg = (double*)(dsm + stage_off) + (size_t)warp * 128 * D;
      for (int k = warp; k < lev_end; k += nwarps) {
        const int i = (int)queue[k];
        const int n = nbn[i], e = nbe[i];
        const uint32_t dn = den[i], cn = ccnt[i];
        const double rd = rden[i];
        const uint4* ls = (const uint4*)(lists + (int64_t)i * KP);
        double num = 0.0;
        for (int t0 = 0; t0 < n; t0 += 128) {
          const int tb = t0 + 4 * lane;
          uint4 r = make_uint4(0u, 0u, 0u, 0u);
          if (tb < n) r = __ldg(&ls[tb >> 2]);
          const uint32_t ent[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
            if (tb + jj > e && tb + jj < n) release_one((int)ent[jj]);
          double v[4][D];
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int cc = 0; cc < D; ++cc)
              v[jj][cc] = (tb + jj < n) ? __ldcg(&Q[(int64_t)ent[jj] * D + cc]) : 0.0;
#pragma unroll
          for (int jj = 0; jj < 4; ++jj)
#pragma unroll
            for (int cc = 0; cc < D; ++cc) stg[(4 * lane + jj) * D + cc] = v[jj][cc];
          __syncwarp();
          if (lane < D && n > 1) {
            const int len = min(128, n - t0);
#pragma unroll 8
            for (int u = 0; u < len; ++u) num = __dadd_rn(num, stg[u * D + lane]);
          }
          __syncwarp();
        }
        if (n > 1 && lane < D) {  // else: frozen or isolated (Q row = S_old, P3)
          const double s1 = gl_div(num, (double)dn, rd);
          __stcg(&Q[((int64_t)P1ROW + i) * D + lane], __dmul_rn((double)cn, s1));
          __stcg(&Q[(int64_t)i * D + lane], s1);
        }
      }
      if (prof) {
        __syncthreads();
        if (pl && tid == 0) pl[2] = clock64();
      }
    } else {
    // ---- update the frontier cells this CTA owns
    for (int base = qhead + warp * CPW; base < lev_end; base += nwarps * CPW) {
      const int k = base + q;
      const bool act = q < CPW && k < lev_end;
      const int i = act ? (int)queue[k] : 0;
      // every load that depends only on i is issued together (nbn, the per-cell scalars, the
      // list words and -- for d <= 3 all, for d > 3 the first block of -- operand rows): the
      // rows beyond the list's end are the zero row (lists are padded to KP), so they need
      // not wait for n
      const int n = act ? nbn[i] : 0;
      const uint32_t dn = act ? den[i] : 1u, cn = act ? ccnt[i] : 0u;
      const double rd = act ? rden[i] : 1.0;
      const uint4* ls = (const uint4*)(lists + (int64_t)i * KP);
      double num = 0.0;
      if constexpr (D <= 3) {
        constexpr int NW = (D == 1 ? 3 : D == 2 ? 9 : 27) / 4 + 1;
        uint4 r[NW];
        double v[NW][4];
        if (act) {
#pragma unroll
          for (int w = 0; w < NW; ++w) r[w] = __ldg(&ls[w]);
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            v[w][0] = __ldcg(&Q[(int64_t)r[w].x * D + c]);
            v[w][1] = __ldcg(&Q[(int64_t)r[w].y * D + c]);
            v[w][2] = __ldcg(&Q[(int64_t)r[w].z * D + c]);
            v[w][3] = __ldcg(&Q[(int64_t)r[w].w * D + c]);
          }
        }
        if (n > 1) {
#pragma unroll
          for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int t = 0; t < 4; ++t) num = __dadd_rn(num, v[w][t]);
        }
      } else {
        constexpr int WB = 4;
        uint4 ra[WB], rb[WB];
        double va[WB][4], vb[WB][4];
        if (act) {  // first block: no dependence on n
#pragma unroll
          for (int w = 0; w < WB; ++w) ra[w] = __ldg(&ls[min(w, KP / 4 - 1)]);
#pragma unroll
          for (int w = 0; w < WB; ++w) {
            va[w][0] = __ldcg(&Q[(int64_t)ra[w].x * D + c]);
            va[w][1] = __ldcg(&Q[(int64_t)ra[w].y * D + c]);
            va[w][2] = __ldcg(&Q[(int64_t)ra[w].z * D + c]);
            va[w][3] = __ldcg(&Q[(int64_t)ra[w].w * D + c]);
          }
        }
        if (n > 1) {
          const int nq = (n + 3) >> 2;
          auto fetch = [&](uint4 (&r)[WB], double (&v)[WB][4], int w0) {
#pragma unroll
            for (int w = 0; w < WB; ++w) r[w] = __ldg(&ls[min(w0 + w, KP / 4 - 1)]);
#pragma unroll
            for (int w = 0; w < WB; ++w) {
              const bool in = w0 + w < nq;
              v[w][0] = in ? __ldcg(&Q[(int64_t)r[w].x * D + c]) : 0.0;
              v[w][1] = in ? __ldcg(&Q[(int64_t)r[w].y * D + c]) : 0.0;
              v[w][2] = in ? __ldcg(&Q[(int64_t)r[w].z * D + c]) : 0.0;
              v[w][3] = in ? __ldcg(&Q[(int64_t)r[w].w * D + c]) : 0.0;
            }
          };
          auto fold = [&](const double (&v)[WB][4]) {
#pragma unroll
            for (int w = 0; w < WB; ++w)
#pragma unroll
              for (int t = 0; t < 4; ++t) num = __dadd_rn(num, v[w][t]);
          };
          for (int w0 = 0; w0 < nq; w0 += 2 * WB) {
            if (w0 + WB < nq) fetch(rb, vb, w0 + WB);
            fold(va);
            if (w0 + WB >= nq) break;
            if (w0 + 2 * WB < nq) fetch(ra, va, w0 + 2 * WB);
            fold(vb);
          }
        }
      }
      if (n > 1) {  // else: frozen or no active neighbour but itself (Q row = S_old, P3)
        const double s1 = gl_div(num, (double)dn, rd);
        __stcg(&Q[((int64_t)P1ROW + i) * D + c], __dmul_rn((double)cn, s1));
        __stcg(&Q[(int64_t)i * D + c], s1);
      }
    }
    if (prof) {
      __syncthreads();
      if (pl && tid == 0) pl[2] = clock64();
    }
    // ---- release the successors into their owners' pending counts / next queues (DSMEM):
    //      a warp per frontier cell, one lane per successor (the remote atomic chains of a
    //      cell's successors run in parallel)
    constexpr int RW = 32;
    for (int k = qhead + tid / RW; k < lev_end; k += T / RW) {
      const int i = (int)queue[k];
      const int n = nbn[i], e = nbe[i];
      const uint32_t* li = lists + (int64_t)i * KP;
      for (int t = e + 1 + (RW == 1 ? 0 : lane); t < n; t += RW) {
        const int j = (int)__ldg(&li[t]);
        const int own = j % NC;
        unsigned* pj = cluster.map_shared_rank(pend + j / NC, own);
        if (atomicSub(pj, 1u) == 1u) {
          unsigned* tl = cluster.map_shared_rank(&tails[nxt], own);
          unsigned* qd = cluster.map_shared_rank(nxt ? qbuf1 : qbuf0, own);
          qd[atomicAdd(tl, 1u)] = (unsigned)j;
        }
      }
    }
    }
    __syncthreads();  // this CTA is done reading queue[cur]
    if (pl && tid == 0) pl[3] = clock64();
    if (tid == 0) {
      tails[cur] = 0u;  // refilled only during the next level, after the barrier
      if (lev_end > 0) atomicAdd(cnt0 + level % 3, (unsigned)lev_end);
    }
    cluster.sync();  // rows, releases and counts of this level are complete and visible
    if (pl && tid == 0) pl[4] = clock64();
    total += *(volatile unsigned*)(cnt0 + level % 3);
    if (rank == 0 && tid == 0) done_cnt[(level + 2) % 3] = 0u;  // everyone read it before this
    ++level;
    if (total >= m) break;
  }
  if (prof && rank == 0 && tid == 0) prof[1000 * 16 * 5] = level;
  cluster.sync();  // no CTA exits while others may still read its shared memory
}

// ---------------------------------------------------------------- dataflow cluster sweep
// The cluster sweep without levels: a cell is updated as soon as its last lex-earlier
// neighbour is, by a warp of its owner CTA that waits on the next position of the owner's
// queue (every owned cell is appended exactly once, after all of its predecessors were
// processed, so a warp waiting on position k only waits for cells at earlier positions of some
// queue: no deadlock).  A warp updates one cell (lane l loads list word l of each 128-entry
// chunk, the operand rows are staged per warp, lanes c < D add them in list order), stores the
// row, and releases the successors with remote atomics on their owners' pending counts; the
// last releaser appends the successor with an atomic on the owner's tail and a store of the
// cell id into the owner's queue slot (initialised to -1; the consumer polls it with an
// acquire load).  Memory ordering (PTX model, cluster scope): after the warp barrier every
// lane -- the row writers included -- executes fence.acq_rel.cluster, so each successor's
// relaxed decrement is a release pattern over the rows; the last releaser's fence after its
// decrement acquires the other releasers' rows through the count's RMW chain and releases them
// with the queue-slot store; the consumer's ld.acquire pairs with it, and a warp barrier
// carries it to the lanes that load the rows.  No barrier, no
// level skew: the critical path is the DAG depth x one update + one release.  A spin watchdog
// sets err bit 8 instead of hanging.  Operands and add order are the serial sweep's.
__device__ __forceinline__ int ld_acquire_cluster_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];"
               : "=r"(v)
               : "r"((uint32_t)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_cluster() {
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}

template <int D>
__host__ __device__ constexpr size_t sweep_flow_smem(int mloc) {
  return (((size_t)8 * mloc + 15) & ~(size_t)15) + (size_t)(512 / 32) * 128 * D * 8;
}

template <int D>
__global__ void __launch_bounds__(512, 1) k_sweep_flow(
    int m, int KP, const uint32_t* __restrict__ lists, const int32_t* __restrict__ nbn,
    const int32_t* __restrict__ nbe, const uint32_t* __restrict__ ccnt,
    const uint32_t* __restrict__ den, const double* __restrict__ rden, double* Q, int* err,
    int flow_sleep, int flow_fence, const int32_t* __restrict__ pinit = nullptr) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int NC = (int)cluster.num_blocks(), rank = (int)cluster.block_rank();
  extern __shared__ __align__(16) unsigned char dsm[];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = T >> 5;
  const int mloc = (m + NC - 1) / NC;
  const int own_n = rank < m ? (m - rank + NC - 1) / NC : 0;  // cells rank, rank+NC, ...
  unsigned* pend = (unsigned*)dsm;
  int* queue = (int*)(pend + mloc);
  double* stg = (double*)(dsm + (((size_t)8 * mloc + 15) & ~(size_t)15)) + (size_t)warp * 128 * D;
  __shared__ unsigned tail;
  if (tid == 0) tail = 0;
  for (int t = tid; t < mloc; t += T) queue[t] = -1;
  __syncthreads();
  for (int t = tid; t < own_n; t += T) {
    const int i = rank + NC * t;
    const int e = pinit ? pinit[i] : nbe[i];  // pending predecessors
    pend[t] = (unsigned)e;
    if (e == 0) queue[atomicAdd(&tail, 1u)] = i;
  }
  const uint32_t P1ROW = (uint32_t)m + 1u;
  cluster.sync();  // every CTA's pending counts and queue slots are initialised
  bool dead = false;
  for (int pos = warp; pos < own_n && !dead; pos += nwarps) {
    int i = -1;
    if (lane == 0) {
      long long spins = 0;
      while ((i = ld_acquire_cluster_s32(&queue[pos])) < 0) {
        if (++spins > (1ll << 26)) {  // watchdog: never hang the GPU
          atomicOr(err, 8);
          break;
        }
        if (flow_sleep) __nanosleep(flow_sleep);
      }
    }
    i = __shfl_sync(0xffffffffu, i, 0);
    __syncwarp();  // lane 0's acquire is ordered before every lane's operand-row loads
    if (i < 0) {
      dead = true;
      break;
    }
    const int n = nbn[i], e = nbe[i];
    const uint32_t dn = den[i], cn = ccnt[i];
    const double rd = rden[i];
    const uint4* ls = (const uint4*)(lists + (int64_t)i * KP);
    double num = 0.0;
    uint32_t ent_keep[4];  // this lane's entries of the last chunk (for the release)
    int tb_keep = 0;
    for (int t0 = 0; t0 < max(n, 1); t0 += 128) {
      const int tb = t0 + 4 * lane;
      uint4 r = make_uint4(0u, 0u, 0u, 0u);
      if (tb < n) r = __ldg(&ls[tb >> 2]);
      const uint32_t ent[4] = {r.x, r.y, r.z, r.w};
      double v[4][D];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int cc = 0; cc < D; ++cc)
          v[jj][cc] = (tb + jj < n) ? __ldcg(&Q[(int64_t)ent[jj] * D + cc]) : 0.0;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
#pragma unroll
        for (int cc = 0; cc < D; ++cc) stg[(4 * lane + jj) * D + cc] = v[jj][cc];
      __syncwarp();
      if (lane < D && n > 1) {
        const int len = min(128, n - t0);
#pragma unroll 8
        for (int u = 0; u < len; ++u) num = __dadd_rn(num, stg[u * D + lane]);
      }
      __syncwarp();
      if (t0 + 128 >= n) {  // the last chunk's words stay in registers for the release
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) ent_keep[jj] = ent[jj];
        tb_keep = tb;
      }
    }
    if (n > 1 && lane < D) {  // else: frozen or isolated (Q row = S_old, P3)
      const double s1 = gl_div(num, (double)dn, rd);
      __stcg(&Q[((int64_t)P1ROW + i) * D + lane], __dmul_rn((double)cn, s1));
      __stcg(&Q[(int64_t)i * D + lane], s1);
    }
    __syncwarp();
    if (flow_fence) __threadfence();  // (diagnostic variant: GPU-scope fence as well)
    fence_acq_rel_cluster();  // every lane: the rows precede any release of a successor
    auto release_one = [&](int j) {
      const int own = j % NC;
      unsigned* pj = cluster.map_shared_rank(pend + j / NC, own);
      if (atomicSub(pj, 1u) == 1u) {
        fence_acq_rel_cluster();  // acquire the other releasers' rows, release them all
        unsigned* tl = cluster.map_shared_rank(&tail, own);
        int* qd = cluster.map_shared_rank(queue, own);
        const unsigned slot = atomicAdd(tl, 1u);  // slot uniqueness only
        atomicExch(&qd[slot], j);
      }
    };
    // successors: entries e < t < n; the last chunk's from registers, earlier chunks reloaded
    for (int t0 = 0; t0 + 128 < n; t0 += 128) {
      const int tb = t0 + 4 * lane;
      const uint4 r = __ldg(&ls[tb >> 2]);
      const uint32_t ent[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int jj = 0; jj < 4; ++jj)
        if (tb + jj > e && tb + jj < n) release_one((int)ent[jj]);
    }
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
      if (tb_keep + jj > e && tb_keep + jj < n) release_one((int)ent_keep[jj]);
  }
  cluster.sync();  // no CTA exits while others may still touch its shared memory
}

// ---------------------------------------------------------------- component sweep (r2)
// Eq. (5)'s sweep couples a cell only to its active neighbours, so the connected components
// of the active cells (adjacency = the 3^d neighbourhood) are swept independently: the
// sequential lexicographic sweep restricted to one component performs exactly the same
// updates, with the same operands in the same order, as the sweep over all cells.  cfg5's
// first iteration has 62 components of <= 4,095 cells and a 125-level DAG; the cluster sweep
// pays ~8.6 K cycles per level (operands in L2, a cluster barrier); here one CTA per component
// holds everything in shared memory and pays one block barrier per level.
//   k_cc_init / k_cc_jump / k_cc_hook / k_cc_count   union-find over each cell's lex-earlier
//                neighbours (the lists of k_nbr_lists) in global memory on all SMs; roots,
//                component sizes and bounding boxes
//   k_cc_plan_par offsets of the components of >= 2 cells, count, largest (block scans + atomics)
//                shared-memory need (cells + bounding box)
//   k_cc_scatter member lists per component (any order: the sweep's result does not depend on
//                the order of a level's cells)
//   k_sweep_comp one CTA per component: the cells' rows (C'*S, replaced by C'*S_new when the
//                cell is updated -- every reader of the old row is a predecessor, finished
//                before), a u16 index over the component's bounding box (+1 margin), per cell
//                its box position, neighbour mask, count and ΣC', the pending counts and two
//                frontier queues, all in shared memory.  Per level, a lane per (cell,
//                coordinate) resolves the active neighbours through the box index in lex
//                offset order (the serial sweep's operands and order, pin P2), divides with
//                RN(1/ΣC') (Markstein), stores S_new to Q's row and C'*S_new to its shared row,
//                then the warp releases the lex-later neighbours (every decrement in flight
//                together, ONE tail atomic per warp); one block barrier per level.  Singleton
//                cells (isolated or frozen) keep the Q row k_nbr_lists wrote (S_old, pin P3).
constexpr int kCcMaxCells = 1 << 20;  // (u16 local indices limit a component, not m)

template <int D>
__host__ __device__ constexpr int comp_K() { return D == 1 ? 3 : D == 2 ? 9 : 27; }

// shared-memory bytes of one component: rows (sz + 1 with the zero row) 8D; per cell its box
// position, C', ΣC' (4 B each), a u16 pending count and a u16 queue slot (20 B); the u16 box
// index (2 B per box cell)
template <int D>
__host__ __device__ constexpr size_t sweep_comp_smem(long long sz, long long box) {
  return (size_t)(sz + 1) * D * 8 + (size_t)sz * 16 + (size_t)((sz + 1) & ~1ll) * 2 +
         (size_t)box * 2 + 64;
}

// Connected components in global memory, all SMs (ECL-CC style): every cell hooked to its
// smallest lex-earlier neighbour (list entry 0: lists are in lex offset order over lex-sorted
// cells), pointer jumping to shorten the chains, then the other lex-earlier neighbours united
// (finds with path halving; a hook puts a root under a smaller root, so pointers only ever go
// to smaller indices and every root ends as its component's smallest cell).
__device__ __forceinline__ int cc_find_g(int32_t* par, int x) {
  int cur = __ldcg(&par[x]);
  if (cur == x) return x;
  int prev = x, nxt;
  while (cur > (nxt = __ldcg(&par[cur]))) {
    __stcg(&par[prev], nxt);
    prev = cur;
    cur = nxt;
  }
  return cur;
}

template <int D>
__global__ void k_cc_init(int m, int KP, const uint32_t* __restrict__ lists,
                          const int32_t* __restrict__ nbe, int32_t* __restrict__ par,
                          int32_t* __restrict__ gsize, int32_t* __restrict__ cur,
                          int32_t* __restrict__ bmin, int32_t* __restrict__ bmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  par[i] = nbe[i] > 0 ? (int)(__ldg(&lists[(int64_t)i * KP]) - ((uint32_t)m + 1u)) : i;
  gsize[i] = 0;
  cur[i] = 0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    bmin[(size_t)i * D + c] = INT_MAX;
    bmax[(size_t)i * D + c] = INT_MIN;
  }
}

__global__ void k_cc_jump(int m, int32_t* par) {  // par[i] <- its great-grandparent
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int p = __ldcg(&par[i]);
  p = __ldcg(&par[p]);
  p = __ldcg(&par[p]);
  __stcg(&par[i], p);
}

template <int D>
__global__ void k_cc_hook(int m, int KP, const uint32_t* __restrict__ lists,
                          const int32_t* __restrict__ nbe, int32_t* par) {
  constexpr int KE = comp_K<D>() / 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int e = nbe[i];
  const uint32_t P1ROW = (uint32_t)m + 1u;
  int jj[KE];
#pragma unroll
  for (int t = 1; t < KE; ++t) jj[t] = t < e ? (int)(__ldg(&lists[(int64_t)i * KP + t]) - P1ROW) : -1;
#pragma unroll
  for (int t = 1; t < KE; ++t) {
    if (jj[t] < 0) continue;
    int a = cc_find_g(par, i), bb = cc_find_g(par, jj[t]);
    while (a != bb) {
      if (a < bb) {
        const int t2 = a;
        a = bb;
        bb = t2;
      }
      const int old = atomicCAS(&par[a], a, bb);
      if (old == a) break;
      a = cc_find_g(par, old);
      bb = cc_find_g(par, bb);
    }
  }
}

// roots; sizes and bounding boxes reduced per group of equal roots in a warp
template <int D>
__global__ void k_cc_count(int m, GsBox b, const uint32_t* __restrict__ ckey, int32_t* par,
                           int32_t* __restrict__ gsize, int32_t* __restrict__ bmin,
                           int32_t* __restrict__ bmax) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = i < m;
  int r = -1, x[D];
  if (in) {
    r = cc_find_g(par, i);
    const uint32_t L = ckey[i] % (uint32_t)b.vol_frame;
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = (int)((L / (uint32_t)b.stride[c]) % (uint32_t)b.ext[c]);
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) x[c] = 0;
  }
  const unsigned g = __match_any_sync(0xffffffffu, r);
  const int n = __popc(g);
  int lo[D], hi[D];
#pragma unroll
  for (int c = 0; c < D; ++c) {
    lo[c] = __reduce_min_sync(g, x[c]);
    hi[c] = __reduce_max_sync(g, x[c]);
  }
  if (in && (int)(threadIdx.x & 31) == __ffs(g) - 1) {
    atomicAdd(&gsize[r], n);
#pragma unroll
    for (int c = 0; c < D; ++c) {
      atomicMin(&bmin[(size_t)r * D + c], lo[c]);
      atomicMax(&bmax[(size_t)r * D + c], hi[c]);
    }
  }
  if (in) __stcg(&par[i], r);  // (roots are final: compress)
}

// The plan: components of >= 2 cells -> coff (per root, -1 otherwise), desc[c] = {offset, size,
// root, -}; ctr[0] = components, ctr[1] = largest size, ctr[2] = largest shared-memory need of
// k_sweep_comp, ctr[3] = its component ticket, ctr[4] = cells in components (the member array's
// fill); ctr is zeroed before the launch.  On all SMs (r2, session 4; one CTA scanning all roots
// took 19 us on cfg5): the offsets only have to be disjoint, not in root order (member lists in
// any order give the same sweep), so every block scans its 256 roots and takes its share of the
// member array and of the descriptor list with two atomics.
template <int D>
__global__ void __launch_bounds__(256) k_cc_plan_par(int m, const int32_t* __restrict__ gsize,
                                                     const int32_t* __restrict__ bmin,
                                                     const int32_t* __restrict__ bmax,
                                                     int32_t* __restrict__ coff,
                                                     int32_t* __restrict__ desc,
                                                     unsigned long long* __restrict__ ctr) {
  __shared__ int s_v[8], s_c[8];
  __shared__ int s_base_off, s_base_c;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int i = blockIdx.x * blockDim.x + tid;
  const int sz = i < m ? gsize[i] : 0;
  const bool comp = sz >= 2;
  long long box = 1;
  if (comp) {
#pragma unroll
    for (int q = 0; q < D; ++q)
      box *= (long long)(bmax[(size_t)i * D + q] - bmin[(size_t)i * D + q] + 3);
  }
  int xv = comp ? sz : 0, xc = comp ? 1 : 0;
  const int v = xv, cf = xc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, xv, o), b2 = __shfl_up_sync(0xffffffffu, xc, o);
    if (lane >= o) {
      xv += a;
      xc += b2;
    }
  }
  if (lane == 31) {
    s_v[wid] = xv;
    s_c[wid] = xc;
  }
  unsigned long long need = comp ? (unsigned long long)sweep_comp_smem<D>(sz, box) : 0ull;
  int mx = comp ? sz : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    need = max(need, __shfl_xor_sync(0xffffffffu, need, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __syncthreads();
  int pv = 0, pc = 0, tv = 0, tc = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    if (w < wid) {
      pv += s_v[w];
      pc += s_c[w];
    }
    tv += s_v[w];
    tc += s_c[w];
  }
  if (tid == 0) {
    s_base_off = tc ? (int)atomicAdd(&ctr[4], (unsigned long long)tv) : 0;
    s_base_c = tc ? (int)atomicAdd(&ctr[0], (unsigned long long)tc) : 0;
  }
  if (lane == 0 && mx) {
    atomicMax(&ctr[1], (unsigned long long)mx);
    atomicMax(&ctr[2], need);
  }
  __syncthreads();
  if (i >= m) return;
  if (!comp) {
    coff[i] = -1;
    return;
  }
  const int off = s_base_off + pv + xv - v, c = s_base_c + pc + xc - cf;
  coff[i] = off;
  desc[4 * c] = off;
  desc[4 * c + 1] = sz;
  desc[4 * c + 2] = i;
  desc[4 * c + 3] = 0;
}

__global__ void k_cc_scatter(int m, const int32_t* __restrict__ root,
                             const int32_t* __restrict__ coff, int32_t* __restrict__ cur,
                             int32_t* __restrict__ mem) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int r = root[i];
  const int o = coff[r];
  if (o < 0) return;
  mem[o + atomicAdd(&cur[r], 1)] = i;
}

template <int D>
__global__ void __launch_bounds__(256) k_sweep_comp(
    int m, GsBox b, const int32_t* __restrict__ desc, const int32_t* __restrict__ mem,
    const int32_t* __restrict__ bmin, const int32_t* __restrict__ bmax,
    const uint32_t* __restrict__ ckey, const uint32_t* __restrict__ ccnt, double* Q,
    long long* __restrict__ plan, long long budget) {
  constexpr int K = comp_K<D>(), KE = K / 2;  // offsets t < KE are lex-earlier, t == KE self
  constexpr int CPW = 32 / D;
  extern __shared__ __align__(16) unsigned char csm[];
  // The plan is read here, not by the host (which reads it while this kernel runs): CTAs take
  // components by ticket; a plan that does not fit a CTA makes the whole launch a no-op and
  // the host, seeing the same plan, runs the cluster sweep instead.
  const long long ncomp = plan[0];
  if (ncomp == 0 || plan[1] >= 65535 || plan[2] > budget) return;
  __shared__ int s_ci;
  for (;;) {
  __syncthreads();  // the previous component's shared state is dead
  if (threadIdx.x == 0) s_ci = (int)atomicAdd((unsigned long long*)&plan[3], 1ull);
  __syncthreads();
  const int ci = s_ci;
  if (ci >= ncomp) return;
  const int off = desc[4 * ci], sz = desc[4 * ci + 1];
  const int r0 = desc[4 * ci + 2];
  int blo[D], bst[D];
  int V = 1;
#pragma unroll
  for (int c = D - 1; c >= 0; --c) {  // the component's box with one empty layer per side
    blo[c] = bmin[(size_t)r0 * D + c] - 1;
    bst[c] = V;
    V *= bmax[(size_t)r0 * D + c] - blo[c] + 2;
  }
  __shared__ int s_offs[K];
  __shared__ unsigned s_cnt[3];  // cells appended by level L live in s_cnt[(L + 1) % 3]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  double* row = (double*)csm;                               // (sz + 1) x D, zero row sz
  uint32_t* bpos = (uint32_t*)(row + (size_t)(sz + 1) * D);  // box position per cell
  uint32_t* cnt = bpos + sz;                                 // C'
  uint32_t* dsum = cnt + sz;                                 // ΣC'
  uint32_t* pend = dsum + sz;                                // u16 pending counts, in pairs
  uint16_t* queue = (uint16_t*)(pend + ((sz + 1) >> 1));     // every cell appended once
  uint16_t* bidx = queue + ((sz + 1) & ~1);                  // box index (0xffff: none)
  if (tid == 0) s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
  for (int t = tid; t < K; t += blockDim.x) {  // lex offsets (dim 0 most significant)
    int r = t, o = 0;
#pragma unroll
    for (int c = D - 1; c >= 0; --c) {
      o += (r % 3 - 1) * bst[c];
      r /= 3;
    }
    s_offs[t] = o;
  }
  for (int t = tid; t < V; t += blockDim.x) bidx[t] = 0xffffu;
  for (int t = tid; t < ((sz + 1) >> 1); t += blockDim.x) pend[t] = 0u;
  __syncthreads();
  for (int l = tid; l < sz; l += blockDim.x) {
    const int g = mem[off + l];
    const int64_t L = (int64_t)(ckey[g] % (uint32_t)b.vol_frame);
    uint32_t p = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) p += (uint32_t)((int)((L / b.stride[c]) % b.ext[c]) - blo[c]) * bst[c];
    bpos[l] = p;
    bidx[p] = (uint16_t)l;
    cnt[l] = ccnt[g];
#pragma unroll
    for (int c = 0; c < D; ++c) row[(size_t)l * D + c] = __ldcg(&Q[(int64_t)g * D + c]);
  }
  if (tid < D) row[(size_t)sz * D + tid] = 0.0;
  __syncthreads();
  for (int l = tid; l < sz; l += blockDim.x) {  // ΣC', pending counts, first frontier
    const uint32_t p = bpos[l];
    uint32_t s = 0;
    int e = 0;
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const uint32_t j = bidx[p + s_offs[t]];
      if (j != 0xffffu) {
        s += cnt[j];
        e += t < KE;
      }
    }
    dsum[l] = s;
    if (e) atomicAdd(&pend[l >> 1], (unsigned)e << (16 * (l & 1)));
    else queue[atomicAdd(&s_cnt[0], 1u)] = (uint16_t)l;
  }
  __syncthreads();
  const int q = lane / D, c = lane - (lane / D) * D;
  int offs[K];  // the lex offsets in registers
#pragma unroll
  for (int t = 0; t < K; ++t) offs[t] = s_offs[t];
  int h0 = 0, t0 = 0;  // the frontier: queue[h0, t0)
  for (int L = 0;; ++L) {
    h0 = t0;
    t0 += (int)*(volatile unsigned*)&s_cnt[L % 3];
    if (h0 == t0) break;
    if (tid == 0) s_cnt[(L + 2) % 3] = 0u;  // its last readers passed the previous barrier
    unsigned* nct = &s_cnt[(L + 1) % 3];
    for (int base = h0 + warp * CPW; base < t0; base += nwarps * CPW) {
      const int k = base + q;
      const bool act = q < CPW && k < t0;
      const int l = act ? (int)queue[k] : sz;
      const uint32_t p = act ? bpos[l] : 0u;
      uint32_t jn[K];
#pragma unroll
      for (int t = 0; t < K; ++t) jn[t] = act ? (uint32_t)bidx[p + offs[t]] : 0xffffu;
      // release the lex-later neighbours first (their updates run after this level's barrier,
      // which orders this cell's row store before them): lane c of the cell takes offsets
      // KE+1+c, +D, ...; every decrement in flight before any result is used
      constexpr int RMAX = (K - KE - 1 + D - 1) / D;
      uint32_t js[RMAX], od[RMAX];
#pragma unroll
      for (int r = 0; r < RMAX; ++r) js[r] = 0xffffu;
#pragma unroll
      for (int t = KE + 1; t < K; ++t)  // (static indices: the lane's share selected by predicate)
        if ((t - KE - 1) % D == c) js[(t - KE - 1) / D] = jn[t];
#pragma unroll
      for (int r = 0; r < RMAX; ++r)
        od[r] = js[r] != 0xffffu
                    ? (atomicSub(&pend[js[r] >> 1], 1u << (16 * (js[r] & 1))) >> (16 * (js[r] & 1))) & 0xffffu
                    : 0u;
      int nr = 0;
#pragma unroll
      for (int r = 0; r < RMAX; ++r) nr += od[r] == 1u;
      if (nr) {
        int at = t0 + (int)atomicAdd(nct, (unsigned)nr);
#pragma unroll
        for (int r = 0; r < RMAX; ++r)
          if (od[r] == 1u) queue[at++] = (uint16_t)js[r];
      }
      if (act) {  // (a component cell always has an active neighbour besides itself)
        const int g = mem[off + l];
        const uint32_t dn = dsum[l], cn = cnt[l];
        const double rd = __drcp_rn((double)dn);
        double t2[K];
#pragma unroll
        for (int t = 0; t < K; ++t) t2[t] = row[(size_t)(jn[t] != 0xffffu ? jn[t] : (uint32_t)sz) * D + c];
        double num = 0.0;
#pragma unroll
        for (int t = 0; t < K; ++t)
          if (jn[t] != 0xffffu) num = __dadd_rn(num, t2[t]);
        const double s1 = gl_div(num, (double)dn, rd);
        Q[(int64_t)g * D + c] = s1;
        row[(size_t)l * D + c] = __dmul_rn((double)cn, s1);
      }
    }
    __syncthreads();
  }
  }  // next component
}

}  // namespace gs
