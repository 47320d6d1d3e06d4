// gs_global.cuh — the sweep of the global path (frames too large for one CTA's smem).
//
// Same design as K8's sweep (gs_resident.cuh), with the cell state in L2-resident global
// memory:
//   k_nbr_count / k_nbr_fill (all SMs)  neighbour census, then per cell {slot, C'} records of
//                                        its lex-earlier active neighbours, the C'*S_old
//                                        products and slots of itself and its lex-later ones,
//                                        ΣC' and RN(1/ΣC')
//   k_sweep_kahn (one CTA)               Kahn frontier over the sweep DAG: each level is
//                                        updated with every operand final, then releases its
//                                        lex-later neighbours
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
  if (!(fa < 0x1p+1000) || (fa < 0x1p-900 && a != 0.0)) return __ddiv_rn(a, b);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}

// One CTA.  pend/queue live in dynamic shared memory when 8*m bytes fit (smem_cells >= m),
// else in the global scratch arrays.
template <int D>
__global__ void __launch_bounds__(1024, 1) k_sweep_kahn(
    int m, int smem_cells, const int32_t* __restrict__ nbn, const int32_t* __restrict__ nbe,
    const int32_t* __restrict__ eoff, const int32_t* __restrict__ loff,
    const unsigned long long* __restrict__ erec, const double* __restrict__ lprod,
    const int32_t* __restrict__ lsucc, const uint32_t* __restrict__ den,
    const double* __restrict__ rden, const double* __restrict__ S0, double* S1, int* pend_g,
    int* queue_g) {
  extern __shared__ int sq[];
  const int tid = threadIdx.x, T = blockDim.x;
  constexpr int CH = D <= 3 ? 8 : 4;
  const bool in_smem = m <= smem_cells;
  volatile int* pend = in_smem ? sq : pend_g;
  volatile int* queue = in_smem ? sq + smem_cells : queue_g;
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
    for (int k = qhead + tid; k < lev_end; k += T) {
      const int i = queue[k];
      const int n = nbn[i], e = nbe[i];
      if (n <= 1) {  // isolated or frozen: centroid kept bit-for-bit (pin P3)
#pragma unroll
        for (int c = 0; c < D; ++c) S1[(int64_t)i * D + c] = S0[(int64_t)i * D + c];
      } else {
        double num[D];
#pragma unroll
        for (int c = 0; c < D; ++c) num[c] = 0.0;
        const unsigned long long* er = erec + eoff[i];
        for (int t0 = 0; t0 < e; t0 += CH) {  // earlier neighbours: NEW centroids
          unsigned long long r[CH];
          double v[CH][D];
#pragma unroll
          for (int u = 0; u < CH; ++u) r[u] = (t0 + u < e) ? er[t0 + u] : 0ull;
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            const int64_t j = (uint32_t)r[u];
#pragma unroll
            for (int c = 0; c < D; ++c) v[u][c] = (t0 + u < e) ? __ldcg(&S1[j * D + c]) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < CH; ++u)
            if (t0 + u < e) {
              const double w = (double)(uint32_t)(r[u] >> 32);
#pragma unroll
              for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], __dmul_rn(w, v[u][c]));
            }
        }
        const double* lp = lprod + (int64_t)loff[i] * D;
        const int nl = n - e;
        for (int t0 = 0; t0 < nl; t0 += CH) {  // itself + later neighbours: C'*S_old
          double v[CH][D];
#pragma unroll
          for (int u = 0; u < CH; ++u)
#pragma unroll
            for (int c = 0; c < D; ++c) v[u][c] = (t0 + u < nl) ? lp[(t0 + u) * D + c] : 0.0;
#pragma unroll
          for (int u = 0; u < CH; ++u)
            if (t0 + u < nl) {
#pragma unroll
              for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], v[u][c]);
            }
        }
        const double dd = (double)den[i], y = rden[i];
#pragma unroll
        for (int c = 0; c < D; ++c) S1[(int64_t)i * D + c] = gl_div(num[c], dd, y);
      }
      // release the lex-later neighbours (self is the first late record)
      const int l0 = loff[i] + 1, ns = n - e - 1;
      for (int t = 0; t < ns; ++t) {
        const int j = lsucc[l0 + t];
        if (atomicSub((int*)&pend[j], 1) == 1) queue[atomicAdd(&tail, 1u)] = j;
      }
    }
    qhead = lev_end;
  }
}

}  // namespace gs
