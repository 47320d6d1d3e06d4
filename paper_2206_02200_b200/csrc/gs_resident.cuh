// gs_resident.cuh — K8: the CTA-resident GridShift iteration engine.
//
// One thread block owns one frame (frames are independent runs) and executes
// the whole engine loop of SPEC.md:135-143 for it with the cell state in shared memory:
//   hash index of the active keys (smem open addressing)
//   -> neighbour lists in lexicographic v order
//   -> Eq. (5) sweep with exact sequential semantics: per-cell dataflow on smem ready-flags
//      (a cell waits only for its lex-earlier active neighbours; SPEC.md:120(b,c))
//   -> rehome floor(S/h), changed / max displacement (SPEC.md:120(d,e), :108)
//   -> bitonic sort of (new key, old rank) and ordered Eq. (3) folds
//   -> root composition for the member sets (Eq. 4), has_converged
// with no global synchronisation and no host round trip per iteration.  Every fp64
// expression is the same _rn sequence as the global-path kernels and the CPU oracle.
#pragma once

#include <cstdint>

#include "gs_common.cuh"

namespace gs {

struct ResidentArgs {
  GsBox box;
  int ms;        // shared-memory cell capacity (power of two)
  int pool_cap;  // neighbour-pool capacity (u16 entries)
  int max_iter;
  int record;
  const uint32_t* ckey;  // current cells (global, frame-major, lex order within a frame)
  const uint32_t* ccnt;
  const double* S;
  const int32_t* ffirst;  // current cell range of each frame
  const int32_t* fcount;
  const int32_t* ifirst;  // initial cell range of each frame (root entries)
  const int32_t* icount;
  int32_t* fdone;
  int32_t* fiters;
  int32_t* fconv;
  int32_t* fk;
  uint32_t* okey;  // final cells, written at the frame's current offset
  uint32_t* ocnt;
  double* oS;
  int32_t* root;  // initial cell -> current cell (global index in, frame-local id out)
  int64_t* hist_m;
  double* hist_d;
  int* err;
};

// shared-memory bytes per cell (excluding the neighbour pool) for dimension D
__host__ __device__ constexpr int resident_bytes_per_cell(int D) {
  return 16 * D /*S0,S1*/ + 8 /*sort key*/ + 16 /*key A/B, cnt A/B*/ + 4 /*den*/ + 4 /*flag*/ +
         16 /*nbn, nbe, nboff, par*/ + 4 /*tmp*/ + 16 /*hash: 2 slots x (key, val)*/;
}

__device__ __forceinline__ uint32_t rs_hash(uint32_t k, int bits) {
  return (k * 2654435761u) >> (32 - bits);
}

__device__ __forceinline__ int rs_lookup(const uint32_t* htk, const int32_t* htv, int bits,
                                         uint32_t k) {
  const uint32_t mask = (1u << bits) - 1u;
  uint32_t h = rs_hash(k, bits);
  for (;;) {
    const uint32_t kk = htk[h];
    if (kk == k) return htv[h];
    if (kk == 0xffffffffu) return -1;
    h = (h + 1) & mask;
  }
}

// Exclusive scan of a[0..n) in shared memory (in place); returns the total.  All threads.
__device__ int rs_scan(int* a, int n, int* wtmp) {
  const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int chunk = (n + T - 1) / T;
  const int beg = min(n, tid * chunk), end = min(n, beg + chunk);
  int local = 0;
  for (int j = beg; j < end; ++j) local += a[j];
  int x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) wtmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    const int nw = T >> 5;
    int w = lane < nw ? wtmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) wtmp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int run = x - local + (wid > 0 ? wtmp[wid - 1] : 0);
  for (int j = beg; j < end; ++j) {
    const int v = a[j];
    a[j] = run;
    run += v;
  }
  const int total = wtmp[(T >> 5) - 1];
  __syncthreads();
  return total;
}

template <int D>
__global__ void __launch_bounds__(1024) k_resident(ResidentArgs a) {
  const GsBox& b = a.box;
  const int f = blockIdx.x;
  const int tid = threadIdx.x, T = blockDim.x;
  const int first = a.ffirst[f];
  int m = a.fcount[f];
  const int ifirst = a.ifirst[f], icnt = a.icount[f];
  const int64_t fbase = (int64_t)f * b.vol_frame;
  int iters = a.fiters[f];
  int conv = a.fconv[f];
  // root entries of this frame: global current index -> frame-local index
  for (int c = ifirst + tid; c < ifirst + icnt; c += T) a.root[c] -= first;
  if (a.fdone[f] || m > a.ms) {
    if (m > a.ms && !a.fdone[f] && tid == 0) atomicOr(a.err, 16);
    for (int i = tid; i < m; i += T) {  // finished in the global path: copy out
      a.okey[first + i] = a.ckey[first + i];
      a.ocnt[first + i] = a.ccnt[first + i];
      for (int c = 0; c < D; ++c) a.oS[(int64_t)(first + i) * D + c] = a.S[(int64_t)(first + i) * D + c];
    }
    if (tid == 0) a.fk[f] = m;
    return;
  }

  // ---- shared-memory carve-up
  extern __shared__ __align__(16) unsigned char smem[];
  const int MS = a.ms;
  unsigned char* p = smem;
  double* S0 = (double*)p;          p += sizeof(double) * MS * D;
  double* S1 = (double*)p;          p += sizeof(double) * MS * D;
  uint64_t* sk = (uint64_t*)p;      p += sizeof(uint64_t) * MS;
  uint32_t* keyA = (uint32_t*)p;    p += 4 * MS;
  uint32_t* keyB = (uint32_t*)p;    p += 4 * MS;
  uint32_t* cntA = (uint32_t*)p;    p += 4 * MS;
  uint32_t* cntB = (uint32_t*)p;    p += 4 * MS;
  uint32_t* den = (uint32_t*)p;     p += 4 * MS;
  uint32_t* flag = (uint32_t*)p;    p += 4 * MS;
  int* nbn = (int*)p;               p += 4 * MS;
  int* nbe = (int*)p;               p += 4 * MS;
  int* nboff = (int*)p;             p += 4 * MS;
  int* par = (int*)p;               p += 4 * MS;
  int* tmp = (int*)p;               p += 4 * MS;
  uint32_t* htk = (uint32_t*)p;     p += 4 * 2 * MS;
  int32_t* htv = (int32_t*)p;       p += 4 * 2 * MS;
  uint16_t* pool = (uint16_t*)p;
  __shared__ int wtmp[32];
  __shared__ unsigned long long s_dmax;
  volatile uint32_t* vflag = flag;

  uint32_t* key = keyA;
  uint32_t* cnt = cntA;
  uint32_t* nkey = keyB;
  uint32_t* ncnt = cntB;

  for (int i = tid; i < m; i += T) {
    key[i] = (uint32_t)((int64_t)a.ckey[first + i] - fbase);
    cnt[i] = a.ccnt[first + i];
    for (int c = 0; c < D; ++c) S0[i * D + c] = a.S[(int64_t)(first + i) * D + c];
    flag[i] = 0u;
  }
  const int K = [] {
    int k = 1;
    for (int c = 0; c < D; ++c) k *= 3;
    return k;
  }();

  auto build_hash = [&](int mm, int& bits) {
    bits = 1;
    while ((1 << bits) < 2 * mm) ++bits;
    const int hs = 1 << bits;
    for (int j = tid; j < hs; j += T) htk[j] = 0xffffffffu;
    __syncthreads();
    const uint32_t mask = (uint32_t)hs - 1u;
    for (int i = tid; i < mm; i += T) {
      uint32_t h = rs_hash(key[i], bits);
      for (;;) {
        const uint32_t prev = atomicCAS(&htk[h], 0xffffffffu, key[i]);
        if (prev == 0xffffffffu) {
          htv[h] = i;
          break;
        }
        h = (h + 1) & mask;
      }
    }
    __syncthreads();
  };

  int bits;
  __syncthreads();
  build_hash(m, bits);

  bool done = false;
  while (!done) {
    const uint32_t epoch = (uint32_t)iters + 1u;
    // ---- (1) neighbour lists: active 1-neighbourhood in lex v order, #earlier, ΣC'
    for (int i = tid; i < m; i += T) {
      GsNbrOdometer od;
      od.init(b);
      int n = 0;
      for (int t = 0; t < K; ++t) {
        n += rs_lookup(htk, htv, bits, (uint32_t)((int64_t)key[i] + od.off)) >= 0;
        od.next(b);
      }
      nbn[i] = n;
      tmp[i] = n;
    }
    __syncthreads();
    const int total = rs_scan(tmp, m, wtmp);
    const bool pooled = total <= a.pool_cap;
    for (int i = tid; i < m; i += T) {
      nboff[i] = tmp[i];
      GsNbrOdometer od;
      od.init(b);
      int e = 0, n = 0;
      uint32_t s = 0;
      for (int t = 0; t < K; ++t) {
        const int j = rs_lookup(htk, htv, bits, (uint32_t)((int64_t)key[i] + od.off));
        if (j >= 0) {
          if (pooled) pool[tmp[i] + n] = (uint16_t)j;
          ++n;
          e += (j < i);
          s += cnt[j];
        }
        od.next(b);
      }
      nbe[i] = e;
      den[i] = s;
    }
    if (tid == 0) s_dmax = 0ull;
    __syncthreads();

    // ---- (2) the sweep: dataflow over the static DAG of this iteration
    for (int base = 0; base < m; base += T) {
      const int i = base + tid;
      bool pending = i < m;
      int n = 0, e = 0, t_ok = 0;
      if (pending) {
        n = nbn[i];
        e = nbe[i];
        if (n <= 1) {  // no active neighbour but itself: centroid kept bit-for-bit (pin P3)
          for (int c = 0; c < D; ++c) S1[i * D + c] = S0[i * D + c];
          __threadfence_block();
          vflag[i] = epoch;
          pending = false;
        }
      }
      if (pooled) {
        const uint16_t* lst = pool + (pending ? nboff[i] : 0);
        while (__any_sync(0xffffffffu, pending)) {
          if (pending) {
            while (t_ok < e && vflag[lst[t_ok]] == epoch) ++t_ok;
            if (t_ok == e) {
              __threadfence_block();
              double num[D];
#pragma unroll
              for (int c = 0; c < D; ++c) num[c] = 0.0;
              for (int t = 0; t < n; ++t) {
                const int j = lst[t];
                const double w = (double)cnt[j];
                const double* src = (t < e) ? S1 : S0;
#pragma unroll
                for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], __dmul_rn(w, src[j * D + c]));
              }
              const double dd = (double)den[i];
#pragma unroll
              for (int c = 0; c < D; ++c) S1[i * D + c] = __ddiv_rn(num[c], dd);
              __threadfence_block();
              vflag[i] = epoch;
              pending = false;
            }
          }
        }
      } else if (pending) {
        // pool overflow (very dense high-d neighbourhoods): look neighbours up again, waiting
        // on each earlier one in turn (independent thread scheduling keeps lanes progressing)
        double num[D];
#pragma unroll
        for (int c = 0; c < D; ++c) num[c] = 0.0;
        GsNbrOdometer od;
        od.init(b);
        for (int t = 0; t < K; ++t) {
          const int j = rs_lookup(htk, htv, bits, (uint32_t)((int64_t)key[i] + od.off));
          od.next(b);
          if (j < 0) continue;
          if (j < i) {
            while (vflag[j] != epoch) {
            }
            __threadfence_block();
          }
          const double w = (double)cnt[j];
          const double* src = (j < i) ? S1 : S0;
#pragma unroll
          for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], __dmul_rn(w, src[j * D + c]));
        }
        const double dd = (double)den[i];
#pragma unroll
        for (int c = 0; c < D; ++c) S1[i * D + c] = __ddiv_rn(num[c], dd);
        __threadfence_block();
        vflag[i] = epoch;
      }
    }
    __syncthreads();

    // ---- (3) rehome, changed, displacement
    int P = 1;
    while (P < m) P <<= 1;
    bool ch = false, bad = false;
    for (int i = tid; i < P; i += T) {
      if (i >= m) {
        sk[i] = ~0ull;
        continue;
      }
      int64_t Ln = 0;
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double s1 = S1[i * D + c], s0 = S0[i * D + c];
        const int64_t rel = gs_grid_coord(s1, b.h, b.inv_h) - b.kmin[c];
        bad |= (rel < 1) | (rel > b.ext[c] - 2);
        Ln += rel * b.stride[c];
        ch |= __double_as_longlong(s1) != __double_as_longlong(s0);
        const double t = __dsub_rn(s1, s0);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
      }
      if (bad) Ln = key[i];
      ch |= (Ln != (int64_t)key[i]);
      atomicMax(&s_dmax, (unsigned long long)__double_as_longlong(__dsqrt_rn(acc)));
      sk[i] = ((uint64_t)(uint32_t)Ln << 32) | (uint32_t)i;
    }
    if (bad) atomicOr(a.err, 4);
    const int changed = __syncthreads_or(ch);
    const double dmax = __longlong_as_double((long long)s_dmax);

    // ---- (4) bitonic sort of (new key, old rank): members of a merge group end up
    //          adjacent and in visit order
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

    // ---- (5) segments -> new cells; parent map
    for (int j = tid; j < m; j += T)
      tmp[j] = (j == 0 || (sk[j] >> 32) != (sk[j - 1] >> 32)) ? 1 : 0;
    __syncthreads();
    const int mnew = rs_scan(tmp, m, wtmp);
    for (int j = tid; j < m; j += T) {
      const bool head = (j == 0 || (sk[j] >> 32) != (sk[j - 1] >> 32));
      const int g = tmp[j] + (head ? 1 : 0) - 1;
      par[(uint32_t)sk[j]] = g;
      if (head) nboff[g] = j;  // segment start (nboff is free after the sweep)
    }
    __syncthreads();
    // merge_into folded in visit order (Eq. 3, pin P4)
    for (int g = tid; g < mnew; g += T) {
      const int start = nboff[g];
      const int end = (g + 1 < mnew) ? nboff[g + 1] : m;
      const uint32_t i0 = (uint32_t)sk[start];
      double s[D];
#pragma unroll
      for (int c = 0; c < D; ++c) s[c] = S1[i0 * D + c];
      uint64_t cc = cnt[i0];
      for (int j = start + 1; j < end; ++j) {
        const uint32_t i = (uint32_t)sk[j];
        const uint64_t ci = cnt[i];
        const double x = (double)cc, w = (double)ci, tot = (double)(cc + ci);
#pragma unroll
        for (int c = 0; c < D; ++c)
          s[c] = __ddiv_rn(__dadd_rn(__dmul_rn(x, s[c]), __dmul_rn(w, S1[i * D + c])), tot);
        cc += ci;
      }
      nkey[g] = (uint32_t)(sk[start] >> 32);
      ncnt[g] = (uint32_t)cc;
#pragma unroll
      for (int c = 0; c < D; ++c) S0[g * D + c] = s[c];
    }
    // member union (Eq. 4) as root composition
    for (int c = ifirst + tid; c < ifirst + icnt; c += T) a.root[c] = par[a.root[c]];
    __syncthreads();
    {
      uint32_t* t1 = key;
      key = nkey;
      nkey = t1;
      uint32_t* t2 = cnt;
      cnt = ncnt;
      ncnt = t2;
    }
    const int m_before = m;
    m = mnew;
    build_hash(m, bits);

    // ---- (6) has_converged on the new state
    bool adj = false;
    for (int i = tid; i < m && !adj; i += T) {
      GsNbrOdometer od;
      od.init(b);
      for (int t = 0; t < K; ++t) {
        if (od.off != 0 && rs_lookup(htk, htv, bits, (uint32_t)((int64_t)key[i] + od.off)) >= 0) {
          adj = true;
          break;
        }
        od.next(b);
      }
    }
    const int any_adj = __syncthreads_or(adj);
    if (tid == 0 && a.record) {
      a.hist_m[(int64_t)f * a.max_iter + iters] = m_before;
      a.hist_d[(int64_t)f * a.max_iter + iters] = dmax;
    }
    ++iters;
    conv = (!any_adj || !changed) ? 1 : 0;
    done = conv || iters >= a.max_iter;
  }

  for (int i = tid; i < m; i += T) {
    a.okey[first + i] = (uint32_t)((int64_t)key[i] + fbase);
    a.ocnt[first + i] = cnt[i];
    for (int c = 0; c < D; ++c) a.oS[(int64_t)(first + i) * D + c] = S0[i * D + c];
  }
  if (tid == 0) {
    a.fk[f] = m;
    a.fiters[f] = iters;
    a.fconv[f] = conv;
    a.fdone[f] = 1;
  }
}

// current cell range of every frame (cells are frame-major)
__global__ void k_frame_ranges(int m, int64_t vol_frame, const uint32_t* __restrict__ key,
                               int32_t* __restrict__ first, int32_t* __restrict__ count) {
  int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= m) return;
  const int64_t f = key[g] / vol_frame;
  if (g == 0 || (int64_t)(key[g - 1] / vol_frame) != f) first[f] = g;
  if (g == m - 1 || (int64_t)(key[g + 1] / vol_frame) != f) count[f] = g + 1;  // end; fixed up
}

__global__ void k_frame_counts(int64_t nf, const int32_t* __restrict__ first,
                               int32_t* __restrict__ count) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f < nf) count[f] -= first[f];
}

// label table from frame-local final ids
__global__ void k_labtab_local(int m0, const uint32_t* __restrict__ initkey,
                               const int32_t* __restrict__ root, int32_t* __restrict__ lab) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m0) lab[initkey[i]] = root[i];
}

}  // namespace gs
