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

#include "gs_common.cuh"

namespace gs {

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

__device__ __forceinline__ double gl_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double fa = fabs(a);
  if (!(fa < 0x1p+1000) || (fa < 0x1p-900 && a != 0.0)) return gs_ddiv_slow(a, b);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
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

}  // namespace gs
