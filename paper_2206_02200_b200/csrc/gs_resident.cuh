// gs_resident.cuh — K8: the CTA-resident GridShift iteration engine.
//
// One thread block owns one frame (frames are independent runs) and executes
// the whole engine loop of SPEC.md:135-143 for it with the cell state in shared memory:
//   dense int16 key index over the frame's key box (or the global grid)
//   -> neighbour lists in lexicographic v order, ΣC' and RN(1/ΣC')
//   -> Eq. (5) sweep with exact sequential semantics as Kahn frontiers over the sweep's DAG
//      (a cell waits only for its lex-earlier active neighbours; SPEC.md:120(b,c)): a schedule
//      warp publishes frontier after frontier, two update warps consume them
//   -> rehome floor(S/h), changed / max displacement (SPEC.md:120(d,e), :108)
//   -> bitonic sort of (new key, old rank) and ordered Eq. (3) folds
//   -> root composition for the member sets (Eq. 4), has_converged
// with no global synchronisation and no host round trip per iteration.  Every fp64
// expression is the same _rn sequence as the global-path kernels and the CPU oracle.
//
// The sweep's critical path is (DAG depth) x (one level's latency on a lone warp); DESIGN.md
// §4 and profiles/r1_k8_sweep_level_probe.txt give the measured cost model it is built for.
#pragma once

#include <cstdint>

#include "gs_common.cuh"

namespace gs {

struct ResidentArgs {
  const GsBox* pbox;  // the run's key box (device: the optimistic path never sees it on the host)
  int ms;          // shared-memory cell capacity (power of two)
  int pool_bytes;  // shared-memory bytes for neighbour records
  int max_iter;
  int record;
  const uint32_t* ckey;  // current cells (global, frame-major, lex order within a frame)
  const uint32_t* ccnt;
  const double* S;
  const int32_t* ffirst;  // first current cell of each frame
  const int32_t* fcount;  // cells per frame, or null: ffirst[f + 1] - ffirst[f]
  const int32_t* ifirst;  // initial cell range of each frame (root entries), nframes + 1
  const uint32_t* initkey;  // initial cell -> its dense key (label table)
  int32_t* lab;             // dense key of an initial cell -> frame-local final id
  int32_t* fdone;
  int32_t* fiters;
  int32_t* fconv;
  int32_t* fk;
  int32_t* fout;    // first final cell of each frame (= ffirst[f])
  int64_t* fswept;  // += active cells summed over this launch's iterations
  uint32_t* okey;  // final cells, written at the frame's current offset
  uint32_t* ocnt;
  double* oS;
  int32_t* root;  // initial cell -> current cell (global index in, frame-local id out)
  int64_t* hist_m;
  double* hist_d;
  int* err;
  int64_t* mode_count;  // [3]: iterations run in fast / list / inline sweep mode (diagnostic)
  long long* prof;      // [8] per-phase SM cycles summed over frames (diagnostic), or null
  // cell index (key -> slot): a dense int16 table over the frame's key box in shared memory
  // when it fits (sidx_bytes > 0), else the engine's global dense grid (int32, clean = -1)
  int32_t* gidx;
  int sidx_bytes;
  // optimistic launch: a frame with more than ms cells raises *deferred and its CTA leaves at
  // once; the host then redoes the whole run on the synchronous path (global path first)
  int deferrable;
  int* deferred;
  long long* trace;  // optional per-level timeline of frame 0's first iteration (diagnostic)
};

// shared-memory bytes per cell (excluding the index and neighbour-record pool)
__host__ __device__ constexpr int resident_bytes_per_cell(int D) {
  return 24 * D /*S0, Q = S1|P1*/ + 8 /*sort key*/ + 16 /*key A/B, cnt A/B*/ + 4 /*den*/ + 8 /*1/den*/ +
         4 /*flag*/ + 16 /*nbn, nbe, eoff, par*/ + 4 /*tmp*/ + 4 /*initial cell -> current*/;
}

// shared-memory bytes of the neighbour-offset table (int32 per offset) for dimension D
__host__ __device__ constexpr int resident_offs_bytes(int D) {
  return D <= 6 ? (((D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : D == 5 ? 243 : 729) *
                    4 + 15) & ~15)
                : 0;
}

// fixed shared-memory bytes besides the per-cell state: Q's zero row (+ one alignment row)
__host__ __device__ constexpr int resident_fixed_bytes(int D) { return 16 * D; }

// RN(a / b) from y = RN(1/b) (precomputed off the critical path): q0 = RN(a*y); the residual
// a - b*q0 is exact in one FMA; RN(q0 + r*y) is the correctly rounded quotient (Markstein's
// theorem; b is a positive integer count here).  Outside the exponent range where the theorem's
// no-underflow/no-overflow premises hold, fall back to the IEEE division.
__device__ __forceinline__ double rs_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double fa = fabs(a);
  if (!(fa < 0x1p+1000) || (fa < 0x1p-900 && a != 0.0)) return gs_ddiv_slow(a, b);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}

// Register odometer over the 3^D neighbour offsets in lexicographic v order (dim 0 most
// significant); D is a compile-time constant so v[] stays in registers.
template <int D>
struct OdoD {
  int8_t v[D];
  int64_t off;
  __device__ __forceinline__ void init(const GsBox& b) {
    off = 0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      v[c] = -1;
      off -= b.stride[c];
    }
  }
  __device__ __forceinline__ void next(const GsBox& b) {
#pragma unroll
    for (int c = D - 1; c >= 0; --c) {
      if (v[c] < 1) {
        ++v[c];
        off += b.stride[c];
        return;
      }
      v[c] = -1;
      off -= 2 * b.stride[c];
    }
  }
};

__device__ __forceinline__ uint32_t rs_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
               : "=r"(v)
               : "r"((uint32_t)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}

__device__ __forceinline__ void rs_st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}

// named barrier over the first n threads (n a multiple of 32), and its OR-reduction form
__device__ __forceinline__ void rs_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int rs_bar_or(int id, int n, int pred) {
  int r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.s32 p, %3, 0;\n bar.red.or.pred q, %1, %2, p;\n"
      " selp.s32 %0, 1, 0, q;\n}"
      : "=r"(r)
      : "r"(id), "r"(n), "r"(pred)
      : "memory");
  return r;
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
__global__ void __launch_bounds__(512, 1) k_resident(ResidentArgs a) {
  __shared__ GsBox sbox;
  __shared__ int s_err0;
  const int f = blockIdx.x;
  const int tid = threadIdx.x, T = blockDim.x;
  if (tid == 0) {
    sbox = *a.pbox;
    s_err0 = *a.err;
  }
  __syncthreads();
  // non-finite input / key box beyond the grid or the int64 range: binning did not run and the
  // box is not valid (the host reports the error; on the optimistic path K8 is already queued)
  if (s_err0 & GS_ERR_SKIP) return;
  const GsBox& b = sbox;
  // dense cell index of this frame: smem int16 table when the host reserved room for this
  // box's frame volume, else the global grid (L2-resident)
  const bool sdense = a.sidx_bytes >= 2 * b.vol_frame;
  const int first = a.ffirst[f];
  int m = a.fcount ? a.fcount[f] : a.ffirst[f + 1] - first;
  if (a.deferrable && m > a.ms && !a.fdone[f]) {
    if (tid == 0) atomicExch(a.deferred, 1);
    return;
  }
  const int ifirst = a.ifirst[f], icnt = a.ifirst[f + 1] - ifirst;
  const int64_t fbase = (int64_t)f * b.vol_frame;
  int iters = a.fiters[f];
  int conv = a.fconv[f];
  if (a.fdone[f] || m > a.ms) {
    // root entries of this frame: global current index -> frame-local index
    for (int c = ifirst + tid; c < ifirst + icnt; c += T) a.root[c] -= first;
    if (m > a.ms && !a.fdone[f] && tid == 0) atomicOr(a.err, 16);
    for (int i = tid; i < m; i += T) {  // finished in the global path: copy out
      a.okey[first + i] = a.ckey[first + i];
      a.ocnt[first + i] = a.ccnt[first + i];
      for (int c = 0; c < D; ++c)
        a.oS[(int64_t)(first + i) * D + c] = a.S[(int64_t)(first + i) * D + c];
      a.gidx[a.ckey[first + i]] = -1;  // clean-grid invariant
    }
    for (int c = ifirst + tid; c < ifirst + icnt; c += T) a.lab[a.initkey[c]] = a.root[c];
    if (tid == 0) {
      a.fk[f] = m;
      a.fout[f] = first;
    }
    return;
  }

  // ---- shared-memory carve-up
  extern __shared__ __align__(16) unsigned char smem[];
  const int MS = a.ms;
  unsigned char* p = smem;
  double* S0 = (double*)p;          p += sizeof(double) * MS * D;
  // Q: rows [0, MS) the new centroids S1 (during the sweep: C'*S_old until a cell is updated),
  // row MS zeros, rows [MS+1, 2MS+1) C'*S_new of updated cells
  double* Q = (double*)p;           p += sizeof(double) * (2 * MS + 2) * D;
  double* S1 = Q;
  const int ZROW = MS, P1ROW = MS + 1;
  double* rden = (double*)p;        p += sizeof(double) * MS;
  uint64_t* sk = (uint64_t*)p;      p += sizeof(uint64_t) * MS;
  uint32_t* keyA = (uint32_t*)p;    p += 4 * MS;
  uint32_t* keyB = (uint32_t*)p;    p += 4 * MS;
  uint32_t* cntA = (uint32_t*)p;    p += 4 * MS;
  uint32_t* cntB = (uint32_t*)p;    p += 4 * MS;
  uint32_t* den = (uint32_t*)p;     p += 4 * MS;
  uint32_t* flag = (uint32_t*)p;    p += 4 * MS;
  int* nbn = (int*)p;               p += 4 * MS;
  int* nbe = (int*)p;               p += 4 * MS;
  int* eoff = (int*)p;              p += 4 * MS;
  int* par = (int*)p;               p += 4 * MS;
  int* tmp = (int*)p;               p += 4 * MS;
  int* rootl = (int*)p;             p += 4 * MS;
  int16_t* sidx = (int16_t*)p;      p += a.sidx_bytes;
  int* offs = (int*)p;              p += resident_offs_bytes(D);
  unsigned char* pool = p;          // a.pool_bytes
  __shared__ int wtmp[32];
  __shared__ unsigned long long s_dmax;
  __shared__ int s_slow;  // a reciprocal division met an operand outside its proven range
  __shared__ int s_dummy[32];  // atomics of idle lanes
  int* levend = eoff;  // sweep: published frontier ends (+1), 0 = not yet
  volatile uint32_t* vflag = flag;

  uint32_t* key = keyA;
  uint32_t* cnt = cntA;
  uint32_t* nkey = keyB;
  uint32_t* ncnt = cntB;

  for (int i = tid; i < m; i += T) {
    key[i] = (uint32_t)((int64_t)a.ckey[first + i] - fbase);
    if (sdense) a.gidx[a.ckey[first + i]] = -1;  // the smem index takes over
    cnt[i] = a.ccnt[first + i];
    for (int c = 0; c < D; ++c) S0[i * D + c] = a.S[(int64_t)(first + i) * D + c];
    flag[i] = 0u;
  }
  // initial cells of this frame -> current frame-local cell (shared memory when they fit)
  // initial cells of a big frame (icnt > MS) keep their map to the K8-entry cells in global
  // memory; the per-iteration composition then runs over the entry cells in shared memory
  // (rootl[x] = current cell of entry cell x) and is applied to the initial cells once, at
  // the end (a per-iteration pass over cfg5's 45 K initial cells cost ~27 K cycles)
  const bool rsm = icnt <= MS;
  const int m_entry = m;
  for (int c = tid; c < icnt; c += T) {
    const int r = a.root[ifirst + c] - first;
    if (rsm)
      rootl[c] = r;
    else
      a.root[ifirst + c] = r;
  }
  if (!rsm)
    for (int x = tid; x < m_entry; x += T) rootl[x] = x;
  constexpr int K = D == 1 ? 3 : D == 2 ? 9 : D == 3 ? 27 : D == 4 ? 81 : D == 5 ? 243 :
                    D == 6 ? 729 : D == 7 ? 2187 : D == 8 ? 6561 : D == 9 ? 19683 :
                    D == 10 ? 59049 : D == 11 ? 177147 : 531441;
  constexpr bool kTable = resident_offs_bytes(D) > 0;
  if (kTable && tid == 0) {  // lexicographic neighbour offsets, linear in the frame box
    OdoD<D> od;
    od.init(b);
    for (int t = 0; t < K; ++t) {
      offs[t] = (int)od.off;
      od.next(b);
    }
  }
  // the offset of neighbour t: table lookup (D <= 6) or a register odometer (D > 6)
  // (d <= 3: from the strides in registers -- t is a constant in the unrolled loops, so each
  // offset folds to a sum of +-strides with no memory access)
  const int st0 = (int)b.stride[0], st1 = D > 1 ? (int)b.stride[1] : 0,
            st2 = D > 2 ? (int)b.stride[2] : 0;
  struct NbrIt {
    OdoD<D> od;
    const int* tbl;
    int s0, s1, s2;
    __device__ __forceinline__ int64_t at(int t) const {
      if constexpr (D == 1) return (int64_t)(t - 1) * s0;
      if constexpr (D == 2) return (int64_t)(t / 3 - 1) * s0 + (t % 3 - 1) * s1;
      if constexpr (D == 3)
        return (int64_t)(t / 9 - 1) * s0 + (t / 3 % 3 - 1) * s1 + (t % 3 - 1) * s2;
      return kTable ? (int64_t)tbl[t] : od.off;
    }
    __device__ __forceinline__ void step(const GsBox& bb) {
      if (!kTable) od.next(bb);
    }
  };
  auto nbr_begin = [&]() {
    NbrIt it;
    it.tbl = offs;
    it.s0 = st0;
    it.s1 = st1;
    it.s2 = st2;
    if (!kTable) it.od.init(b);
    return it;
  };

  // dense cell index of this frame: smem int16 table or the global grid (L2-resident)
  int32_t* gidx = a.gidx + fbase;
  auto idx_get = [&](int64_t L) -> int { return sdense ? (int)sidx[L] : gidx[L]; };
  auto idx_put = [&](int64_t L, int v) {
    if (sdense)
      sidx[L] = (int16_t)v;
    else
      gidx[L] = v;
  };
  if (sdense)
    for (int j = tid; j < (int)b.vol_frame; j += T) sidx[j] = -1;
  __syncthreads();
  for (int i = tid; i < m; i += T) idx_put(key[i], i);
  __syncthreads();

  // d > 3 with small frames: neighbours by pairwise comparison of byte-packed cell coordinates
  // (|dk| <= 1 in every byte: two __vabsdiffu4) instead of 3^d index probes, which go to the
  // global grid when the frame's box is too large for the shared-memory index (cfg3: 243 L2
  // probes per cell).  Cells are lex-sorted, so ascending j is the lex neighbour order.
  bool pairwise_ok = D > 3 && D <= 8;
#pragma unroll
  for (int c = 0; c < D; ++c) pairwise_ok = pairwise_ok && b.ext[c] <= 256;
  auto pack_cells = [&](int mm) {  // sk[i] = byte-packed coordinates of cell i
    for (int i = tid; i < mm; i += T) {
      const uint32_t L = key[i];
      uint64_t pk = 0;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const uint32_t rel = (L / (uint32_t)b.stride[c]) % (uint32_t)b.ext[c];
        pk |= (uint64_t)rel << (8 * c);
      }
      sk[i] = pk;
    }
  };
  auto near = [](uint64_t x, uint64_t y) {
    const uint32_t d0 = __vabsdiffu4((uint32_t)x, (uint32_t)y);
    const uint32_t d1 = __vabsdiffu4((uint32_t)(x >> 32), (uint32_t)(y >> 32));
    return ((d0 | d1) & 0xfefefefeu) == 0u;
  };

  bool done = false;
  int64_t swept = 0;
  long long t_prev = clock64();
  auto lap = [&](int ph) {
    if (a.trace && tid == 0 && f == 0 && iters < 64) {  // per-iteration phase timeline
      long long* tr = a.trace + 4096 + 8 * iters;
      tr[ph] = clock64();
      if (ph == 0) tr[6] = m;
    }
    if (a.prof && tid == 0) {
      const long long t = clock64();
      atomicAdd((unsigned long long*)&a.prof[ph], (unsigned long long)(t - t_prev));
      t_prev = t;
    }
  };
  auto stamp = [&](int k) {  // diagnostics (GS_TRACE_LEVELS): thread 0 sub-phase stamps
    if (a.trace && tid == 0 && f == 0 && iters < 64) a.trace[9700 + 16 * iters + k] = clock64();
  };
  lap(7);
  while (!done) {
    if (a.trace && tid == 0 && f == 0 && iters < 64) a.trace[4096 + 8 * iters + 7] = clock64();
    const uint32_t epoch = (uint32_t)iters + 1u;
    // ---- (1) neighbour lists: per cell the Q-row of every active neighbour in lex order
    // (C'*S_new rows for lex-earlier ones, C'*S_old rows for itself and later ones), #active,
    // #earlier, the denominator ΣC' and its reciprocal, and Q row i = C'*S_old.
    //   mode 0 (d <= 3, lists fit at a fixed stride of KP entries): one neighbourhood pass,
    //          lists padded with the zero row (the sweep reads them without bounds)
    //   mode 1: census, scan, then lists padded to whole 4-entry words
    //   mode 2: no lists (they do not fit): the sweep looks neighbours up itself
    constexpr int KP = (K + 3) & ~3;
    uint16_t* lst = (uint16_t*)pool;
    auto finish_cell = [&](int i, int n, uint32_t s, bool lists) {
      if (lists) {
        const double ci = (double)cnt[i];
#pragma unroll
        for (int c = 0; c < D; ++c)  // Q row i = C'*S_old until the cell is updated
          Q[i * D + c] = n <= 1 ? S0[i * D + c] : __dmul_rn(ci, S0[i * D + c]);
      }
      den[i] = s;
      rden[i] = __drcp_rn((double)s);  // for rs_div on the sweep's critical path
      levend[i] = 0;
    };
    int mode, n_all = 0;
    stamp(0);
    if (D <= 3 && 2 * KP * m + 16 <= a.pool_bytes) {
      mode = 0;
      for (int i = tid; i < m; i += T) {
        NbrIt it = nbr_begin();
        int n = 0, e = 0;
        uint32_t s = 0;
        const int64_t Li = key[i];
        uint16_t* li = lst + i * KP;
        // branch-free: all 27 index loads (the index kind hoisted out of the loop), then all
        // count loads, then unconditional list stores at the running position (a dropped
        // entry is overwritten by the next one or by the padding).  With a branch per probe
        // a lone warp paid ~100 cycles per neighbour (~3 K cycles per iteration).
        int jn[K];
        if (sdense) {
#pragma unroll
          for (int t = 0; t < K; ++t) jn[t] = sidx[Li + it.at(t)];
        } else {
#pragma unroll
          for (int t = 0; t < K; ++t) jn[t] = gidx[Li + it.at(t)];
        }
        uint32_t cn[K];
#pragma unroll
        for (int t = 0; t < K; ++t) cn[t] = cnt[jn[t] >= 0 ? jn[t] : 0];
#pragma unroll
        for (int t = 0; t < K; ++t) {
          const int j = jn[t];
          const bool ok = j >= 0;
          s += ok ? cn[t] : 0u;
          li[n] = (uint16_t)(j < i ? P1ROW + j : j);
          n += ok ? 1 : 0;
          e += (ok && j < i) ? 1 : 0;
        }
#pragma unroll
        for (int t = 1; t < KP; ++t)  // (entry 0 is the cell itself or an earlier neighbour)
          if (t >= n) li[t] = (uint16_t)ZROW;
        nbn[i] = n;
        nbe[i] = e;
        tmp[i] = i * KP;
        par[i] = ((i * KP + e + 1) << 5) | (n - e - 1);  // later neighbours: first entry, count
        finish_cell(i, n, s, true);
      }
    } else {
      // census and fill with the index kind hoisted out of the probe loops (a branch per probe
      // serialised d = 5's 243 L2 probes: ~110 K cycles per cell when the frame's index is the
      // global grid) and, in the fill, the probes of a batch issued before its list stores
      constexpr int KB = K < 27 ? K : 27;
      auto census = [&](const auto* ix) {
        for (int i = tid; i < m; i += T) {
          NbrIt it = nbr_begin();
          int n = 0, e = 0;
          const int64_t Li = key[i];
#pragma unroll 27
          for (int t = 0; t < K; ++t) {
            const int j = (int)ix[Li + it.at(t)];
            n += (j >= 0);
            e += (j >= 0) & (j < i);
            it.step(b);
          }
          nbn[i] = n;
          nbe[i] = e;
          tmp[i] = (n + 3) & ~3;  // list length padded to whole 4-entry words
        }
      };
      const bool pw = pairwise_ok && m <= T;
      if (pw) {
        pack_cells(m);
        __syncthreads();
        for (int i = tid; i < m; i += T) {
          const uint64_t pi = sk[i];
          int n = 0, e = 0;
          for (int j = 0; j < m; ++j) {
            const bool nb = near(pi, sk[j]);
            n += nb;
            e += nb & (j < i);
          }
          nbn[i] = n;
          nbe[i] = e;
          tmp[i] = (n + 3) & ~3;
        }
      } else if (sdense) {
        census(sidx);
      } else {
        census(gidx);
      }
      __syncthreads();
      n_all = rs_scan(tmp, m, wtmp);
      mode = (2 * n_all + 8 <= a.pool_bytes) ? 1 : 2;
      auto fill = [&](const auto* ix) {
        for (int i = tid; i < m; i += T) {
          NbrIt it = nbr_begin();
          int nn = 0;
          uint32_t s = 0;
          const int64_t Li = key[i];
          uint16_t* li = lst + tmp[i];
          if constexpr (kTable) {
            for (int t0 = 0; t0 < K; t0 += KB) {
              int jb[KB];
#pragma unroll
              for (int u = 0; u < KB; ++u) jb[u] = (int)ix[Li + it.at(t0 + u)];
#pragma unroll
              for (int u = 0; u < KB; ++u) {
                const int j = jb[u];
                if (j < 0) continue;
                s += cnt[j];
                if (mode == 1) li[nn++] = (uint16_t)(j < i ? P1ROW + j : j);
              }
            }
          } else {
            for (int t = 0; t < K; ++t) {
              const int j = (int)ix[Li + it.at(t)];
              it.step(b);
              if (j < 0) continue;
              s += cnt[j];
              if (mode == 1) li[nn++] = (uint16_t)(j < i ? P1ROW + j : j);
            }
          }
          if (mode == 1)
            for (; nn & 3; ++nn) li[nn] = (uint16_t)ZROW;
          finish_cell(i, nbn[i], s, mode == 1);
        }
      };
      if (pw) {
        for (int i = tid; i < m; i += T) {
          const uint64_t pi = sk[i];
          int nn = 0;
          uint32_t s = 0;
          uint16_t* li = lst + tmp[i];
          for (int j = 0; j < m; ++j) {
            if (!near(pi, sk[j])) continue;
            s += cnt[j];
            if (mode == 1) li[nn++] = (uint16_t)(j < i ? P1ROW + j : j);
          }
          if (mode == 1)
            for (; nn & 3; ++nn) li[nn] = (uint16_t)ZROW;
          finish_cell(i, nbn[i], s, mode == 1);
        }
      } else if (sdense) {
        fill(sidx);
      } else {
        fill(gidx);
      }
      if (mode == 1 && tid < 4) lst[n_all + tid] = (uint16_t)ZROW;  // slack word (prefetch)
    }
    stamp(1);
    for (int c = tid; c < D; c += T) Q[ZROW * D + c] = 0.0;
    if (tid == 0) {
      s_dmax = 0ull;
      s_slow = 0;
      if (a.mode_count) atomicAdd((unsigned long long*)&a.mode_count[mode], 1ull);
    }
    __syncthreads();
    lap(0);

    // ---- (2) the sweep: Kahn frontiers over the sweep's DAG (a cell waits for its lex-earlier
    // active neighbours only).  The frontier schedule depends on the graph, not on the values,
    // so warp 1 computes it (pending counts, successor release, one published frontier end per
    // level) running ahead of the two update warps, which consume it.  Each update lane sums
    // its cell's terms in lex order over exactly the serial sweep's operands, read as Q rows:
    // C'*S_new of an earlier neighbour (P1, written by its updater), C'*S_old of itself / a
    // later neighbour (P0, in place until that cell is updated -- all its readers precede it),
    // +0.0 for padding (an exact identity: the running sum is never -0.0).  Bit-identical to
    // the serial sweep.
    // Cost model (measured, B200, one warp per SMSP): every dependent shared-memory round trip,
    // taken branch or barrier costs ~30-120 cycles, so a level's critical path is kept to
    // "barrier -> reload the operands the previous level wrote -> add chain -> divide -> store";
    // the next level's cells, list words and static operands are loaded before the barrier.
    if (mode != 2) {
      const int warp = tid >> 5, lane = tid & 31;
      const unsigned lt = (1u << lane) - 1u;
      int* queue = (int*)sk;  // frontier after frontier
      if (warp == 1) {
        int* pend = (int*)flag;  // lex-earlier active neighbours not yet released
        int qtail = 0;
        for (int base = 0; base < m; base += 32) {
          const int i = base + lane;
          const bool ready = i < m && nbe[i] == 0;
          if (i < m) pend[i] = nbe[i];
          const unsigned mk = __ballot_sync(0xffffffffu, ready);
          if (ready) queue[qtail + __popc(mk & lt)] = i;
          qtail += __popc(mk);
        }
        constexpr int RB = 8;  // successor releases issued together
        int qhead = 0, lev = 0;
        while (qhead < qtail) {
          const int lev_end = qtail;
          __syncwarp();  // the frontier's queue entries are written (and ordered before...)
          if (lane == 0) rs_st_release((uint32_t*)&levend[lev], (uint32_t)lev_end + 1u);  // ...this
          ++lev;
          for (int base = qhead; base < lev_end; base += 32) {
            const int k = base + lane;
            const bool act = k < lev_end;
            const int i = act ? queue[k] : 0;
            int so, ns;  // first later-neighbour entry and their count
            if (D <= 3 && mode == 0) {
              const int dsc = par[i];
              so = dsc >> 5;
              ns = act ? (dsc & 31) : 0;
            } else {
              const int e = nbe[i];
              so = tmp[i] + e + 1;
              ns = act ? nbn[i] - e - 1 : 0;
            }
            const int mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)ns);
            for (int t0 = 0; t0 < mx; t0 += RB) {
              int jj[RB], old[RB];
#pragma unroll
              for (int u = 0; u < RB; ++u) {  // unconditional loads (padding keeps them in the pool)
                const int j = (int)lst[so + (t0 + u < ns ? t0 + u : 0)];
                jj[u] = (t0 + u < ns) ? j : -1;
              }
#pragma unroll
              for (int u = 0; u < RB; ++u) {  // idle lanes add 0 to their own dummy word
                int* tgt = jj[u] >= 0 ? &pend[jj[u]] : &s_dummy[lane];
                old[u] = atomicAdd(tgt, jj[u] >= 0 ? -1 : 0);
              }
              unsigned mk[RB];
#pragma unroll
              for (int u = 0; u < RB; ++u) mk[u] = __ballot_sync(0xffffffffu, jj[u] >= 0 && old[u] == 1);
#pragma unroll
              for (int u = 0; u < RB; ++u) {
                if ((mk[u] >> lane) & 1u) queue[qtail + __popc(mk[u] & lt)] = jj[u];
                qtail += __popc(mk[u]);
              }
            }
          }
          qhead = lev_end;
        }
      } else if (warp == 0 || warp == 2) {
        // update warps (SMSPs 0 and 2): one lane per (cell, coordinate), so every fp64
        // instruction a warp issues carries up to 32/D cells
        constexpr int CPW = 32 / D;  // cells per warp and round
        const int u = warp >> 1, q = lane / D, c = lane - q * D;
        const bool trace = a.trace && f == 0 && tid == 0 && iters == 0;
        int qhead = 0, lev = 0;
        while (qhead < m) {
          long long tt1 = 0;
          int v;
          long long spins = 0;  // watchdog: a schedule that stops short is a bug, not a hang
          while ((v = (int)rs_ld_acquire((const uint32_t*)&levend[lev])) == 0) {
            if (++spins > (1ll << 26)) break;
          }
          if (v == 0) {
            if (lane == 0) atomicOr(a.err, 8);
            break;
          }
          if (trace) tt1 = clock64();
          const int lev_end = v - 1;
          for (int base = qhead + u * CPW; base < lev_end; base += 2 * CPW) {
            const int k = base + q;
            const bool act = q < CPW && k < lev_end;
            const int i = act ? queue[k] : 0;
            const int n = act ? nbn[i] : 0;
            const double ci = (double)cnt[i], dd = (double)den[i], y = rden[i];
            double num = 0.0;
            auto fetch = [&](double (&vv)[4], uint2 w) {
              vv[0] = Q[(w.x & 0xffffu) * D + c];
              vv[1] = Q[(w.x >> 16) * D + c];
              vv[2] = Q[(w.y & 0xffffu) * D + c];
              vv[3] = Q[(w.y >> 16) * D + c];
            };
            auto fold = [&](const double (&vv)[4]) {
#pragma unroll
              for (int t = 0; t < 4; ++t) num = __dadd_rn(num, vv[t]);
            };
            if constexpr (D <= 3) {
              if (mode == 0) {
                // every word and operand loaded up front, then ONE uniform jump into an
                // unrolled add chain of the warp's longest list (shorter lists add zero rows)
                constexpr int NW = KP / 4;
                const int nchm = (int)__reduce_max_sync(0xffffffffu, (unsigned)((n + 3) >> 2));
                const uint2* ls = (const uint2*)(lst + i * KP);
                const uint2 zw = make_uint2((uint32_t)ZROW * 0x10001u, (uint32_t)ZROW * 0x10001u);
                double vv[NW][4];
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                  const int x = w + nchm - NW;  // slot w holds word w + nchm - NW
                  fetch(vv[w], x >= 0 ? ls[x >= 0 ? x : 0] : zw);
                }
                switch (NW - nchm) {
#define GS_FOLD_SLOT(W)               \
  case W:                             \
    if constexpr (NW > W) fold(vv[W]); \
    [[fallthrough]];
                  GS_FOLD_SLOT(0) GS_FOLD_SLOT(1) GS_FOLD_SLOT(2) GS_FOLD_SLOT(3)
                  GS_FOLD_SLOT(4) GS_FOLD_SLOT(5) GS_FOLD_SLOT(6)
#undef GS_FOLD_SLOT
                  default:
                    break;
                }
              }
            }
            if (mode == 1 && n > 1) {
              const uint2* ls = (const uint2*)(lst + tmp[i]);
              const int nch = (n + 3) >> 2;
              double va[4], vb[4];
              fetch(va, ls[0]);
              for (int ch = 0; ch < nch; ch += 2) {  // next word in flight during the adds
                fetch(vb, ls[ch + 1]);
                fold(va);
                if (ch + 1 >= nch) break;
                fetch(va, ls[ch + 2]);
                fold(vb);
              }
            }
            // RN(num / ΣC') from the precomputed reciprocal; the rare operands outside the
            // theorem's range take the IEEE division (one warp-uniform test)
            const double q0 = __dmul_rn(num, y);
            const double fa = fabs(num);
            const bool slow = !(fa < 0x1p+1000) || (fa < 0x1p-900 && num != 0.0);
            double s1 = __fma_rn(__fma_rn(-q0, dd, num), y, q0);
            if (__any_sync(0xffffffffu, slow && act && n > 1))
              if (slow) s1 = gs_ddiv_slow(num, dd);
            if (act && n > 1) {  // else: no active neighbour but itself, Q row i = S_old (P3)
              Q[(P1ROW + i) * D + c] = __dmul_rn(ci, s1);
              Q[i * D + c] = s1;
            }
          }
          rs_bar(1, 64);  // both update warps: this level's rows are visible to the next level
          if (trace) {
            long long* tr = a.trace + 8 * min(lev, 511);
            tr[0] = 0;
            tr[1] = clock64() - tt1;  // the level
            tr[3] = lev_end - qhead;  // level width
            tr[2] = tr[4] = tr[5] = tr[6] = tr[7] = 0;
          }
          qhead = lev_end;
          ++lev;
        }
      }
      __syncthreads();
    }
    if (mode == 2 || s_slow) {
      // records do not fit (very dense high-d neighbourhoods), or a reciprocal division of the
      // pipelined sweep met an operand outside its proven range (then this recomputes every
      // centroid of the sweep): dataflow with lookups, waiting on each earlier neighbour in
      // turn (independent thread scheduling keeps lanes going)
      for (int i = tid; i < m; i += T) {
        double num[D];
#pragma unroll
        for (int c = 0; c < D; ++c) num[c] = 0.0;
        const int n = nbn[i];
        if (n <= 1) {
#pragma unroll
          for (int c = 0; c < D; ++c) S1[i * D + c] = S0[i * D + c];
        } else {
          NbrIt it = nbr_begin();
          const int64_t Li = key[i];
          for (int t = 0; t < K; ++t) {
            const int j = idx_get(Li + it.at(t));
            it.step(b);
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
          for (int c = 0; c < D; ++c) S1[i * D + c] = rs_div(num[c], dd, rden[i]);
        }
        __threadfence_block();
        vflag[i] = epoch;
      }
      __syncthreads();
    }

    if (a.prof && tid == 0 && iters == 0)  // the first sweep alone (its DAG is data-fixed)
      atomicAdd((unsigned long long*)&a.prof[6], (unsigned long long)(clock64() - t_prev));
    lap(1);
    // ---- (3) rehome, changed, displacement (the displacement only feeds the history)
    int P = 1;
    while (P < m) P <<= 1;
    bool ch = false, bad = false;
    unsigned long long dmx = 0ull;  // |S1 - S0| bits (non-negative doubles order as integers)
    for (int i = tid; i < P; i += T) {
      if (i >= m) {
        sk[i] = ~0ull;
        continue;
      }
      int64_t Ln = 0;
      double acc = 0.0;
      bool bad_i = false;
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double s1 = S1[i * D + c], s0 = S0[i * D + c];
        const int64_t rel = gs_grid_coord(s1, b.h, b.inv_h) - b.kmin[c];
        bad_i |= (rel < 1) | (rel > b.ext[c] - 2);
        Ln += rel * b.stride[c];
        ch |= __double_as_longlong(s1) != __double_as_longlong(s0);
        if (a.record) {
          const double t = __dsub_rn(s1, s0);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
      }
      if (bad_i) Ln = key[i];
      bad |= bad_i;
      ch |= (Ln != (int64_t)key[i]);
      if (a.record) dmx = max(dmx, (unsigned long long)__double_as_longlong(__dsqrt_rn(acc)));
      sk[i] = ((uint64_t)(uint32_t)Ln << 32) | (uint32_t)i;
    }
    if (a.record) {  // one shared atomic per warp
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dmx = max(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
      if ((tid & 31) == 0 && dmx) atomicMax(&s_dmax, dmx);
    }
    if (bad) atomicOr(a.err, 4);
    const int changed = __syncthreads_or(ch);
    const double dmax = __longlong_as_double((long long)s_dmax);
    lap(2);

    // ---- (4) bitonic sort of (new key, old rank): members of a merge group end up
    //          adjacent and in visit order.  With P <= T every thread holds one element:
    //          partners closer than a warp are exchanged by shuffles, farther ones through
    //          two shared buffers (one barrier per such stage).
    uint64_t* sk2 = (uint64_t*)pool;  // the lists are dead after the sweep
    if (P <= T && 8 * P <= a.pool_bytes) {
      uint64_t x = tid < P ? sk[tid] : ~0ull;
      int buf = 0;
      for (int k2 = 2; k2 <= P; k2 <<= 1) {
        for (int j = k2 >> 1; j > 0; j >>= 1) {
          uint64_t y;
          if (j >= 32) {
            uint64_t* bb = buf ? sk2 : sk;
            if (tid < P) bb[tid] = x;
            __syncthreads();
            y = tid < P ? bb[tid ^ j] : ~0ull;
            buf ^= 1;
          } else {
            y = __shfl_xor_sync(0xffffffffu, x, j);
          }
          const bool asc = (tid & k2) == 0, lower = (tid & j) == 0;
          x = (lower == asc) ? min(x, y) : max(x, y);
        }
      }
      if (tid < P) sk[tid] = x;
      __syncthreads();
    } else {
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
    }

    lap(3);
    // ---- (5) segments -> new cells; parent map
    int mnew;
    stamp(2);
    if (m <= T) {  // heads are 0/1: the group ids from one ballot per warp, one barrier
      const int j = tid;
      const bool head = j < m && (j == 0 || (sk[j] >> 32) != (sk[j - 1] >> 32));
      const unsigned bm = __ballot_sync(0xffffffffu, head);
      const int wex = __popc(bm & ((1u << (tid & 31)) - 1u));
      if ((tid & 31) == 0) wtmp[tid >> 5] = __popc(bm);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < (T >> 5); ++w) {
        const int cw = wtmp[w];
        before += (w < (tid >> 5)) ? cw : 0;
        tot += cw;
      }
      mnew = tot;
      if (j < m) {
        const int g = before + wex + (head ? 1 : 0) - 1;
        par[(uint32_t)sk[j]] = g;
        if (head) eoff[g] = j;  // segment start (eoff is free after the sweep)
      }
    } else {
      for (int j = tid; j < m; j += T)
        tmp[j] = (j == 0 || (sk[j] >> 32) != (sk[j - 1] >> 32)) ? 1 : 0;
      __syncthreads();
      mnew = rs_scan(tmp, m, wtmp);
      for (int j = tid; j < m; j += T) {
        const bool head = (j == 0 || (sk[j] >> 32) != (sk[j - 1] >> 32));
        const int g = tmp[j] + (head ? 1 : 0) - 1;
        par[(uint32_t)sk[j]] = g;
        if (head) eoff[g] = j;  // segment start (eoff is free after the sweep)
      }
    }
    stamp(3);
    __syncthreads();
    stamp(4);
    // merge_into folded in visit order (Eq. 3, pin P4): s = RN(RN(RN(x*s) + RN(w*S_i)) / tot),
    // the division from RN(1/tot) (Markstein; the reciprocal does not depend on s, so it
    // leaves the chain); an operand outside the theorem's range redoes the group exactly
    for (int g = tid; g < mnew; g += T) {
      const int start = eoff[g];
      const int end = (g + 1 < mnew) ? eoff[g + 1] : m;
      const uint32_t i0 = (uint32_t)sk[start];
      double s[D];
#pragma unroll
      for (int c = 0; c < D; ++c) s[c] = S1[i0 * D + c];
      uint64_t cc = cnt[i0];
      bool slow = false;
      for (int j = start + 1; j < end; ++j) {
        const uint32_t i = (uint32_t)sk[j];
        const uint64_t ci = cnt[i];
        const double x = (double)cc, w = (double)ci, tot = (double)(cc + ci);
        const double y = __drcp_rn(tot);
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double num = __dadd_rn(__dmul_rn(x, s[c]), __dmul_rn(w, S1[i * D + c]));
          const double fa = fabs(num);
          slow |= !(fa < 0x1p+1000) || (fa < 0x1p-900 && num != 0.0);
          const double q0 = __dmul_rn(num, y);
          s[c] = __fma_rn(__fma_rn(-q0, tot, num), y, q0);
        }
        cc += ci;
      }
      if (slow) {  // rare: the same fold with IEEE divisions
        cc = cnt[i0];
#pragma unroll
        for (int c = 0; c < D; ++c) s[c] = S1[i0 * D + c];
        for (int j = start + 1; j < end; ++j) {
          const uint32_t i = (uint32_t)sk[j];
          const uint64_t ci = cnt[i];
          const double x = (double)cc, w = (double)ci, tot = (double)(cc + ci);
#pragma unroll
          for (int c = 0; c < D; ++c)
            s[c] = gs_ddiv_slow(__dadd_rn(__dmul_rn(x, s[c]), __dmul_rn(w, S1[i * D + c])), tot);
          cc += ci;
        }
      }
      nkey[g] = (uint32_t)(sk[start] >> 32);
      ncnt[g] = (uint32_t)cc;
#pragma unroll
      for (int c = 0; c < D; ++c) S0[g * D + c] = s[c];
    }
    stamp(5);
    // member union (Eq. 4) as root composition
    for (int c = tid; c < (rsm ? icnt : m_entry); c += T) rootl[c] = par[rootl[c]];
    for (int i = tid; i < m; i += T) idx_put(key[i], -1);  // retire the old keys
    stamp(6);
    __syncthreads();
    stamp(7);
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
    lap(4);
    for (int i = tid; i < m; i += T) idx_put(key[i], i);
    __syncthreads();

    // ---- (6) has_converged on the new state
    bool adj = false;
    if (pairwise_ok && m <= T) {
      pack_cells(m);
      __syncthreads();
      for (int i = tid; i < m && !adj; i += T) {
        const uint64_t pi = sk[i];
        for (int j = 0; j < m && !adj; ++j) adj = j != i && near(pi, sk[j]);
      }
    } else
    for (int i = tid; i < m && !adj; i += T) {
      NbrIt it = nbr_begin();
      const int64_t Li = key[i];
      int hits = 0;
      if (sdense) {  // the index kind hoisted: no branch per probe
#pragma unroll 27
        for (int t = 0; t < K; ++t) {
          hits += (t != (K - 1) / 2) && sidx[Li + it.at(t)] >= 0;
          it.step(b);
        }
      } else {
#pragma unroll 27
        for (int t = 0; t < K; ++t) {
          hits += (t != (K - 1) / 2) && gidx[Li + it.at(t)] >= 0;
          it.step(b);
        }
      }
      adj = hits > 0;
    }
    const int any_adj = __syncthreads_or(adj);
    if (tid == 0) {
      swept += m_before;
      if (a.record) {
        a.hist_m[(int64_t)f * a.max_iter + iters] = m_before;
        a.hist_d[(int64_t)f * a.max_iter + iters] = dmax;
      }
    }
    lap(5);
    ++iters;
    conv = (!any_adj || !changed) ? 1 : 0;
    done = conv || iters >= a.max_iter;
  }

  for (int i = tid; i < m; i += T) {
    a.okey[first + i] = (uint32_t)((int64_t)key[i] + fbase);
    a.ocnt[first + i] = cnt[i];
    for (int c = 0; c < D; ++c) a.oS[(int64_t)(first + i) * D + c] = S0[i * D + c];
    if (!sdense) gidx[key[i]] = -1;  // clean-grid invariant for the next run
  }
  for (int c = tid; c < icnt; c += T) {
    int r;
    if (rsm) {
      r = rootl[c];
    } else {
      r = rootl[a.root[ifirst + c]];
      a.root[ifirst + c] = r;
    }
    a.lab[a.initkey[ifirst + c]] = r;
  }
  if (tid == 0) {
    a.fk[f] = m;
    a.fiters[f] = iters;
    a.fconv[f] = conv;
    a.fdone[f] = 1;
    a.fout[f] = first;
    a.fswept[f] += swept;
  }
}

// current cell range of every frame (cells are frame-major)
__global__ void k_frame_ranges(int m, int64_t vol_frame, const uint32_t* __restrict__ key,
                               int32_t* __restrict__ first, int32_t* __restrict__ count,
                               const int32_t* __restrict__ m_dev = nullptr) {
  if (m_dev) m = *m_dev;
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

// End of a global-path iteration: frame cell counts (k_frame_counts), then everything the host
// loop reads, packed for ONE device->host copy -- [mnew, err, -, -] then per frame changed,
// adjacent, swept cells, cell count (int32 each) and the max displacement bits (u64) -- and the
// per-iteration accumulators cleared for the next iteration.
__global__ void k_iter_pack(int64_t nf, const int32_t* __restrict__ first, int32_t* __restrict__ count,
                            int32_t* __restrict__ fchanged, int32_t* __restrict__ fadj,
                            int32_t* __restrict__ fm, unsigned long long* __restrict__ fdisp,
                            const int32_t* __restrict__ mnew_dev, const int* __restrict__ err,
                            int32_t* __restrict__ out) {
  int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (f == 0) {
    out[0] = *mnew_dev;
    out[1] = *err;
  }
  if (f >= nf) return;
  const int32_t c = count[f] - first[f];
  count[f] = c;
  int32_t* o = out + 4;
  o[f] = fchanged[f];
  o[nf + f] = fadj[f];
  o[2 * nf + f] = fm[f];
  o[3 * nf + f] = c;
  ((unsigned long long*)(o + 4 * nf))[f] = fdisp[f];
  fchanged[f] = 0;
  fadj[f] = 0;
  fm[f] = 0;
  fdisp[f] = 0ull;
}


}  // namespace gs
