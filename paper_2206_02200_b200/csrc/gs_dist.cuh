// gs_dist.cuh — multi-GPU drivers of the engine (gridshift_c.h gs_dist_*),
// one host thread driving R ranks, each an engine context on its own device (a device may be
// repeated: loopback ranks on one GPU, used by the tests -- the ranks' kernels never wait on
// each other, every exchange is ordered by the host).  Included at the end of gs_engine.cu
// (it drives the engine's internal kernels and buffers).
//
//  * gs_dist_run_frames: independent frames (cfg4) in contiguous blocks per rank, one host
//    thread per rank, no exchange.
//  * gs_dist_run_slabs: ONE cloud (cfg5) whose points are split into R contiguous shards.
//    Cells are owned by dim-0 slabs of the global key box (cut points balance the initial
//    cells).  Setup: every rank bins its shard into exact partial cells of the global box
//    (integer counts and fixed-point sums); the partial cells go to their slab's owner, which
//    merges them into its initial cells -- bit-identical to one GPU binning the whole cloud.
//    Per iteration (the global path's kernels on each rank's slab):
//      1. halo up: each rank's FIRST key layer (old centroids, as C'*S rows) goes to the rank
//         below;
//      2. sweep, rank by rank in slab order: rank r runs the Kahn sweep over its own cells
//         with the layers of its neighbours frozen in the neighbour lists -- the lower one
//         already swept (rank r-1's LAST layer, C'*S_new rows, sent after r-1's sweep), the
//         upper one not yet (C'*S_old): exactly the single-GPU in-place sweep (Eq. 5), since
//         dim 0 is the most significant key digit, every cell of slab r-1 precedes every cell
//         of slab r;
//      3. rehome: cells whose new key leaves the slab migrate to the owning rank; every rank
//         folds its members (own cells that stay + arrivals) in old global lex order (ranks
//         in slab order, then old local order): Eq. 3's visit order;
//      4. has_converged over the new cells with the neighbours' new boundary keys; `changed`
//         and the max displacement reduced over ranks.
//    The parent map of every iteration is composed on the host into the root of each initial
//    cell (ids = global lexicographic ranks: slab offsets + local ranks), and each rank labels
//    its own points.  All per-iteration data moves are device-to-device peer copies
//    (cudaMemcpyPeerAsync: NVLink between GPUs, a device copy for loopback ranks); the host
//    reads back only keys, counts and parent maps (O(m) words) to plan the exchanges.

#include <thread>

struct gs_dist {
  int R = 0;
  std::vector<int> dev;
  std::vector<gs_ctx*> ctx;
  std::string err;
  bool have_run = false;
  int d = 0;
  int64_t nframes = 0;
  std::vector<int64_t> k;          // clusters per frame
  std::vector<double> cent;        // all frames' centroids, frame after frame
  std::vector<int64_t> cent_off;   // rows before each frame
  std::vector<int64_t> hist_m;     // slabs: active cells per iteration (all ranks)
  std::vector<double> hist_d;      // slabs: max displacement per iteration
  // slab scratch per rank
  struct Rank {
    DevBuf hh_key, hh_cnt, hh_rows, hl_key, hl_cnt, hl_rows, out_rows, mem_idx, mem_key,
        mem_cnt, mem_rows, nkey, bkey, tmp;
  };
  std::vector<Rank> rk;
};

namespace {

gs_status dist_fail(gs_dist* D, gs_status s, const std::string& msg) {
  if (D) D->err = msg;
  return s;
}

#define GS_DCK(call)                                                              \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      D->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
      return (e_ == cudaErrorMemoryAllocation) ? GS_E_OOM : GS_E_CUDA;            \
    }                                                                             \
  } while (0)

#define GS_DTRY(r, expr)                                                          \
  do {                                                                            \
    gs_status s_ = (expr);                                                        \
    if (s_ != GS_OK) {                                                            \
      D->err = "rank " + std::to_string(r) + ": " + D->ctx[r]->err;               \
      return s_;                                                                  \
    }                                                                             \
  } while (0)

// rows[i] = C'_i * S_i (the Q row of a cell that is a later neighbour: k_nbr_lists' product)
__global__ void k_scale_rows(int m, int d, const uint32_t* __restrict__ cnt,
                             const double* __restrict__ S, double* __restrict__ rows) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  for (int c = 0; c < d; ++c)
    rows[(int64_t)i * d + c] = __dmul_rn((double)cnt[i], S[(int64_t)i * d + c]);
}

// members leaving or staying: gather (new key, count, swept row) of the listed old cells
__global__ void k_gather_members(int k, int d, const int32_t* __restrict__ idx,
                                 const uint32_t* __restrict__ nkey,
                                 const uint32_t* __restrict__ cnt, const double* __restrict__ S1,
                                 uint32_t* __restrict__ okey, uint32_t* __restrict__ ocnt,
                                 double* __restrict__ orows) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= k) return;
  const int i = idx[t];
  okey[t] = nkey[i];
  ocnt[t] = cnt[i];
  for (int c = 0; c < d; ++c) orows[(int64_t)t * d + c] = S1[(int64_t)i * d + c];
}

// idx entries for neighbour-slab boundary keys (has_converged probes them, value irrelevant)
__global__ void k_idx_mark(int m, const uint32_t* __restrict__ key, int32_t* __restrict__ idx,
                           int32_t v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) idx[key[i]] = v;
}

// the label table for every initial cell: lab[initial key] = final global id
__global__ void k_lab_scatter(int64_t m, const uint32_t* __restrict__ key,
                              const int32_t* __restrict__ id, int32_t* __restrict__ lab) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) lab[key[i]] = id[i];
}

gs_status peer_copy(gs_dist* D, int dst, void* dptr, int src, const void* sptr, size_t bytes) {
  if (!bytes) return GS_OK;
  GS_DCK(cudaSetDevice(D->dev[dst]));
  GS_DCK(cudaMemcpyPeerAsync(dptr, D->dev[dst], sptr, D->dev[src], bytes, D->ctx[dst]->stream));
  return GS_OK;
}

gs_status rank_sync(gs_dist* D, int r) {
  GS_DCK(cudaSetDevice(D->dev[r]));
  GS_DCK(cudaStreamSynchronize(D->ctx[r]->stream));
  return GS_OK;
}

// dim-0 relative key (box coordinates, apron included) of a linear key of the global box
inline int64_t key_j0(const GsBox& b, uint32_t L) { return (int64_t)L / b.stride[0]; }

// cells [0, a) have j0 == lo, cells [bb, m) have j0 == hi - 1 (keys lex-sorted, dim 0 slowest)
void layer_ranges(const GsBox& b, const std::vector<uint32_t>& keys, int64_t lo, int64_t hi,
                  int64_t* a, int64_t* bb) {
  const int64_t m = (int64_t)keys.size();
  int64_t x = 0;
  while (x < m && key_j0(b, keys[x]) == lo) ++x;
  int64_t y = m;
  while (y > 0 && key_j0(b, keys[y - 1]) == hi - 1) --y;
  *a = x;
  *bb = y;
}

gs_status slab_run(gs_dist* D, const gs_input* in, const gs_config* cfg, gs_result* out) {
  const int R = D->R, d = in->d;
  const int64_t n = in->n;
  const double h = cfg->h;
  const bool rec = (cfg->flags & GS_RECORD_HISTORY) != 0;
  const size_t pb = input_bytes(in) / (size_t)n;  // bytes per point
  std::vector<int64_t> p0(R), pc(R);
  for (int r = 0; r < R; ++r) {
    const int64_t base = n / R, rem = n % R;
    p0[r] = r * base + std::min<int64_t>(r, rem);
    pc[r] = base + (r < rem ? 1 : 0);
    if (pc[r] < 1) return dist_fail(D, GS_E_INVALID_PARAMETER, "fewer points than ranks");
  }
  auto shard = [&](int r) {
    gs_input s = *in;
    s.points = static_cast<const char*>(in->points) + (size_t)p0[r] * pb;
    s.n = pc[r];
    return s;
  };
  // ---- 1. global key box (all-reduce of the shards' key bounds), partial cells per shard
  std::vector<int64_t> klo(d, INT64_MAX), khi(d, INT64_MIN);
  for (int r = 0; r < R; ++r) {
    std::vector<int64_t> lo(d), hi(d);
    const gs_input s = shard(r);
    GS_DTRY(r, gs_shard_keybounds(D->ctx[r], &s, h, lo.data(), hi.data()));
    for (int c = 0; c < d; ++c) {
      klo[c] = std::min(klo[c], lo[c]);
      khi[c] = std::max(khi[c], hi[c]);
    }
  }
  std::vector<std::vector<uint32_t>> pk(R), pcn(R);
  std::vector<std::vector<int64_t>> ps(R);
  for (int r = 0; r < R; ++r) {
    const gs_input s = shard(r);
    int64_t m = 0;
    gs_shard_bin(D->ctx[r], &s, h, n, klo.data(), khi.data(), 0, &m, nullptr, nullptr, nullptr);
    pk[r].resize(m);
    pcn[r].resize(m);
    ps[r].resize((size_t)m * d);
    GS_DTRY(r, gs_shard_bin(D->ctx[r], &s, h, n, klo.data(), khi.data(), m, &m, pk[r].data(),
                            pcn[r].data(), ps[r].data()));
  }
  const GsBox box = D->ctx[0]->box;  // identical on every rank (same bounds, same n)
  // ---- 2. slabs: dim-0 cut points balancing the partial cells (a proxy for the cells)
  const int64_t J = box.ext[0];
  std::vector<int64_t> hist(J, 0);
  for (int r = 0; r < R; ++r)
    for (uint32_t L : pk[r]) hist[key_j0(box, L)]++;
  int64_t tot = 0;
  for (int64_t v : hist) tot += v;
  // cut r ends at the first layer where the cumulative count reaches (r+1)/R of the cells;
  // every slab keeps at least one layer, so two slabs are never adjacent across an empty one
  std::vector<int64_t> lo(R), hi(R);
  {
    std::vector<int64_t> cum(J + 1, 0);
    for (int64_t j = 0; j < J; ++j) cum[j + 1] = cum[j] + hist[j];
    int64_t j = 0;
    for (int r = 0; r < R; ++r) {
      lo[r] = j;
      if (r == R - 1) {
        hi[r] = J;
        break;
      }
      const int64_t target = cum[J] * (r + 1) / R;
      int64_t c = j + 1;
      while (c < J && cum[c] < target) ++c;
      c = std::min<int64_t>(std::max<int64_t>(c, lo[r] + 1), J - (R - 1 - r));
      hi[r] = c;
      j = c;
    }
  }
  // ---- 3. each owner merges the partial cells of its slab into its initial cells
  std::vector<int64_t> m_r(R);
  std::vector<std::vector<uint32_t>> okeys(R), ocnts(R);
  std::vector<std::vector<int64_t>> osums(R);
  for (int src = 0; src < R; ++src)
    for (size_t i = 0; i < pk[src].size(); ++i) {
      const int64_t j0 = key_j0(box, pk[src][i]);
      int dst = 0;
      while (dst < R - 1 && j0 >= hi[dst]) ++dst;
      okeys[dst].push_back(pk[src][i]);
      ocnts[dst].push_back(pcn[src][i]);
      osums[dst].insert(osums[dst].end(), ps[src].begin() + (int64_t)i * d,
                        ps[src].begin() + (int64_t)(i + 1) * d);
    }
  std::vector<uint32_t> init_key;  // every initial cell's key, global id order
  std::vector<int64_t> off(R + 1, 0);
  int64_t npart = 0;  // bounds every later cell count (cells only merge)
  for (int r = 0; r < R; ++r) npart += (int64_t)pk[r].size();
  for (int r = 0; r < R; ++r) {
    gs_ctx* c = D->ctx[r];
    GS_DCK(cudaSetDevice(D->dev[r]));
    // cell buffers sized once for the whole run: a later grow would drop the slab's state
    GS_DTRY(r, ensure_cells(c, npart + 2, d));
    c->shard_m = (int64_t)okeys[r].size();
    c->shard_keys = okeys[r].data();
    c->shard_counts = ocnts[r].data();
    c->shard_sums = osums[r].data();
    c->ev_mask = 0;
    c->cur = 0;
    GS_DTRY(r, ensure_frames(c, 1));
    if (c->shard_m > 0) {
      GS_DTRY(r, launch_shard_front(c, d));
      unsigned ctr[16];
      GS_DCK(cudaMemcpyAsync(ctr, c->counters.p, 64, cudaMemcpyDeviceToHost, c->stream));
      GS_DCK(cudaStreamSynchronize(c->stream));
      m_r[r] = ctr[0];
    } else {
      m_r[r] = 0;
    }
    c->shard_keys = nullptr;
    c->shard_counts = nullptr;
    c->shard_sums = nullptr;
    c->ctl_clean = false;
    std::vector<uint32_t> k0(m_r[r]);
    if (m_r[r])
      GS_DCK(cudaMemcpy(k0.data(), c->ckey[0].p, 4 * m_r[r], cudaMemcpyDeviceToHost));
    init_key.insert(init_key.end(), k0.begin(), k0.end());
    off[r + 1] = off[r] + m_r[r];
  }
  const int64_t m0 = off[R];
  std::vector<int32_t> root(m0);
  for (int64_t i = 0; i < m0; ++i) root[i] = (int32_t)i;
  D->hist_m.clear();
  D->hist_d.clear();
  const int K = (int)ipow3(d);
  // ---- 4. iterations (do-while)
  int iter = 0;
  bool conv = false;
  std::vector<std::vector<uint32_t>> hkeys(R);
  for (;;) {
    for (int r = 0; r < R; ++r) {
      gs_ctx* c = D->ctx[r];
      hkeys[r].resize(m_r[r]);
      GS_DCK(cudaSetDevice(D->dev[r]));
      if (m_r[r])
        GS_DCK(cudaMemcpy(hkeys[r].data(), c->ckey[c->cur].p, 4 * m_r[r], cudaMemcpyDeviceToHost));
    }
    int64_t mt = 0;
    for (int r = 0; r < R; ++r) mt += m_r[r];
    std::vector<int64_t> fa(R), lb(R);  // first layer [0, fa), last layer [lb, m)
    for (int r = 0; r < R; ++r) layer_ranges(box, hkeys[r], lo[r], hi[r], &fa[r], &lb[r]);
    // (1) halo up: rank r+1's first layer (C'*S_old rows) -> rank r
    std::vector<int64_t> nhh(R, 0), nhl(R, 0);
    for (int r = 0; r + 1 < R; ++r) {
      const int s = r + 1;
      gs_ctx* cs = D->ctx[s];
      const int64_t k = fa[s];
      nhh[r] = k;
      if (!k) continue;
      auto& RS = D->rk[s];
      auto& RR = D->rk[r];
      GS_DCK(cudaSetDevice(D->dev[s]));
      GS_DTRY(s, grow(cs, RS.out_rows, 8 * (size_t)k * d));
      k_scale_rows<<<blocks_for(k, 256), 256, 0, cs->stream>>>(
          (int)k, d, cs->ccnt[cs->cur].as<uint32_t>(), cs->S[cs->cur].as<double>(),
          RS.out_rows.as<double>());
      GS_DCK(cudaGetLastError());
      GS_DTRY(s, rank_sync(D, s));
      GS_DCK(cudaSetDevice(D->dev[r]));
      GS_DTRY(r, grow(D->ctx[r], RR.hh_key, 4 * (size_t)k));
      GS_DTRY(r, grow(D->ctx[r], RR.hh_cnt, 4 * (size_t)k));
      GS_DTRY(r, grow(D->ctx[r], RR.hh_rows, 8 * (size_t)k * d));
      GS_DTRY(r, peer_copy(D, r, RR.hh_key.p, s, cs->ckey[cs->cur].p, 4 * k));
      GS_DTRY(r, peer_copy(D, r, RR.hh_cnt.p, s, cs->ccnt[cs->cur].p, 4 * k));
      GS_DTRY(r, peer_copy(D, r, RR.hh_rows.p, s, RS.out_rows.p, 8 * (size_t)k * d));
    }
    // (2) the sweep, slab after slab
    std::vector<int> own_base(R, 0);  // combined index of the first own cell
    std::vector<double*> Qown(R, nullptr);
    for (int r = 0; r < R; ++r) {
      gs_ctx* c = D->ctx[r];
      auto& RR = D->rk[r];
      GS_DCK(cudaSetDevice(D->dev[r]));
      cudaStream_t st = c->stream;
      const int64_t hl = nhl[r], m = m_r[r], hh = nhh[r], mc = hl + m + hh;
      own_base[r] = (int)hl;
      if (m == 0) continue;
      GS_DTRY(r, ensure_cells(c, mc + 1, d));
      const int own = c->cur, cmb = 1 - own;
      // combined cells [lower halo | own | upper halo] in the other buffer
      auto cp = [&](void* dst, const void* src, size_t bytes) -> gs_status {
        if (bytes) GS_DCK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
        return GS_OK;
      };
      GS_DTRY(r, cp(c->ckey[cmb].as<uint32_t>(), RR.hl_key.p, 4 * hl));
      GS_DTRY(r, cp(c->ccnt[cmb].as<uint32_t>(), RR.hl_cnt.p, 4 * hl));
      GS_DTRY(r, cp(c->ckey[cmb].as<uint32_t>() + hl, c->ckey[own].p, 4 * m));
      GS_DTRY(r, cp(c->ccnt[cmb].as<uint32_t>() + hl, c->ccnt[own].p, 4 * m));
      GS_DTRY(r, cp(c->S[cmb].as<double>() + hl * d, c->S[own].p, 8 * m * d));
      GS_DTRY(r, cp(c->ckey[cmb].as<uint32_t>() + hl + m, RR.hh_key.p, 4 * hh));
      GS_DTRY(r, cp(c->ccnt[cmb].as<uint32_t>() + hl + m, RR.hh_cnt.p, 4 * hh));
      GS_DCK(cudaMemsetAsync(c->fdone.p, 0, 4, st));
      GS_DCK(cudaMemsetAsync(c->fm.p, 0, 4, st));
      gs::k_idx_set<<<blocks_for(mc, 256), 256, 0, st>>>((int)mc, c->ckey[cmb].as<uint32_t>(),
                                                        c->idx.as<int32_t>());
      GS_DCK(cudaGetLastError());
      // neighbour lists with the halos frozen, the halo rows the sweep reads, the sweep
      c->cur = cmb;
      c->box = box;
      double* Q = nullptr;
      SweepHalo halo;
      halo.own_lo = (int)hl;
      halo.own_hi = (int)(hl + m);
      halo.rows = [&](double* q) -> gs_status {
        Q = q;
        GS_TRY(cp(q + (hl + m) * d, RR.hh_rows.p, 8 * hh * d));  // upper layer: C'*S_old
        GS_TRY(cp(q + (mc + 1) * d, RR.hl_rows.p, 8 * hl * d));  // lower layer: C'*S_new
        return GS_OK;
      };
      GS_DTRY(r, launch_global_sweep(c, d, mc, K, &halo));
      int err = 0;
      GS_DTRY(r, read_err(c, &err));
      if (err & 8) return dist_fail(D, GS_E_INTERNAL_INVARIANT, "sweep watchdog fired");
      c->cur = own;
      Qown[r] = Q + hl * d;
      // own last layer (C'*S_new rows) -> the next rank's lower halo
      if (r + 1 < R) {
        const int64_t k = m - lb[r];
        nhl[r + 1] = k;
        if (k) {
          auto& RN = D->rk[r + 1];
          gs_ctx* cn = D->ctx[r + 1];
          GS_DCK(cudaSetDevice(D->dev[r + 1]));
          GS_DTRY(r + 1, grow(cn, RN.hl_key, 4 * (size_t)k));
          GS_DTRY(r + 1, grow(cn, RN.hl_cnt, 4 * (size_t)k));
          GS_DTRY(r + 1, grow(cn, RN.hl_rows, 8 * (size_t)k * d));
          GS_DTRY(r + 1, peer_copy(D, r + 1, RN.hl_key.p, r, c->ckey[own].as<uint32_t>() + lb[r], 4 * k));
          GS_DTRY(r + 1, peer_copy(D, r + 1, RN.hl_cnt.p, r, c->ccnt[own].as<uint32_t>() + lb[r], 4 * k));
          GS_DTRY(r + 1, peer_copy(D, r + 1, RN.hl_rows.p, r, Q + (mc + 1 + hl + lb[r]) * d,
                                   8 * (size_t)k * d));
          GS_DTRY(r + 1, rank_sync(D, r + 1));
        }
      }
    }
    // (3) rehome (new keys, `changed`, displacement) on every rank, then the migration plan
    int any_changed = 0;
    double maxdisp = 0.0;
    std::vector<std::vector<uint32_t>> nk(R);
    for (int r = 0; r < R; ++r) {
      gs_ctx* c = D->ctx[r];
      const int64_t m = m_r[r];
      nk[r].resize(m);
      if (!m) continue;
      GS_DCK(cudaSetDevice(D->dev[r]));
      cudaStream_t st = c->stream;
      GS_DCK(cudaMemsetAsync(c->fchanged.p, 0, 4, st));
      GS_DCK(cudaMemsetAsync(c->fdisp.p, 0, 8, st));
      gs::k_rehome<<<blocks_for(m, 256), 256, 0, st>>>(
          (int)m, box, c->ckey[c->cur].as<uint32_t>(), c->S[c->cur].as<double>(), Qown[r],
          c->fdone.as<int32_t>(), c->nkey.as<uint32_t>(), c->vals.as<uint32_t>(),
          c->fchanged.as<int32_t>(), c->fdisp.as<unsigned long long>(), c->errflag.as<int>());
      GS_DCK(cudaGetLastError());
      int32_t ch = 0;
      unsigned long long fd = 0;
      GS_DCK(cudaMemcpyAsync(nk[r].data(), c->nkey.p, 4 * m, cudaMemcpyDeviceToHost, st));
      GS_DCK(cudaMemcpyAsync(&ch, c->fchanged.p, 4, cudaMemcpyDeviceToHost, st));
      GS_DCK(cudaMemcpyAsync(&fd, c->fdisp.p, 8, cudaMemcpyDeviceToHost, st));
      int err = 0;
      GS_DTRY(r, read_err(c, &err));
      if (err & 4) return dist_fail(D, GS_E_INTERNAL_INVARIANT, "centroid left the key box");
      any_changed |= ch;
      double dsp;
      std::memcpy(&dsp, &fd, 8);
      maxdisp = std::max(maxdisp, dsp);
    }
    // members of each destination rank, in old global order: source ranks in slab order,
    // then old local order (Eq. 3's visit order)
    std::vector<std::vector<std::vector<int32_t>>> go(R, std::vector<std::vector<int32_t>>(R));
    for (int s = 0; s < R; ++s)
      for (int64_t i = 0; i < m_r[s]; ++i) {
        const int64_t j0 = key_j0(box, nk[s][i]);
        int dst = 0;
        while (dst < R - 1 && j0 >= hi[dst]) ++dst;
        go[s][dst].push_back((int32_t)i);
      }
    std::vector<int64_t> M(R, 0), mnew(R, 0);
    std::vector<std::vector<int32_t>> parent_local(R);
    std::vector<std::vector<int64_t>> mem_old(R);  // members' old global ids
    for (int dst = 0; dst < R; ++dst)
      for (int s = 0; s < R; ++s) {
        M[dst] += (int64_t)go[s][dst].size();
        for (int32_t i : go[s][dst]) mem_old[dst].push_back(off[s] + i);
      }
    // gather on the sources, copy to the destinations' member arrays
    for (int dst = 0; dst < R; ++dst) {
      gs_ctx* cd = D->ctx[dst];
      auto& RD = D->rk[dst];
      GS_DCK(cudaSetDevice(D->dev[dst]));
      const int64_t Mm = std::max<int64_t>(M[dst], 1);
      GS_DTRY(dst, grow(cd, RD.mem_key, 4 * (size_t)Mm));
      GS_DTRY(dst, grow(cd, RD.mem_cnt, 4 * (size_t)Mm));
      GS_DTRY(dst, grow(cd, RD.mem_rows, 8 * (size_t)Mm * d));
      int64_t pos = 0;
      for (int s = 0; s < R; ++s) {
        const int64_t k = (int64_t)go[s][dst].size();
        if (!k) continue;
        gs_ctx* cs = D->ctx[s];
        auto& RS = D->rk[s];
        GS_DCK(cudaSetDevice(D->dev[s]));
        GS_DTRY(s, grow(cs, RS.mem_idx, 4 * (size_t)k));
        GS_DTRY(s, grow(cs, RS.nkey, 4 * (size_t)k));
        GS_DTRY(s, grow(cs, RS.bkey, 4 * (size_t)k));
        GS_DTRY(s, grow(cs, RS.tmp, 8 * (size_t)k * d));
        GS_DCK(cudaMemcpyAsync(RS.mem_idx.p, go[s][dst].data(), 4 * k, cudaMemcpyHostToDevice,
                               cs->stream));
        k_gather_members<<<blocks_for(k, 256), 256, 0, cs->stream>>>(
            (int)k, d, RS.mem_idx.as<int32_t>(), cs->nkey.as<uint32_t>(),
            cs->ccnt[cs->cur].as<uint32_t>(), Qown[s], RS.nkey.as<uint32_t>(),
            RS.bkey.as<uint32_t>(), RS.tmp.as<double>());
        GS_DCK(cudaGetLastError());
        GS_DTRY(s, rank_sync(D, s));
        GS_DTRY(dst, peer_copy(D, dst, RD.mem_key.as<uint32_t>() + pos, s, RS.nkey.p, 4 * k));
        GS_DTRY(dst, peer_copy(D, dst, RD.mem_cnt.as<uint32_t>() + pos, s, RS.bkey.p, 4 * k));
        GS_DTRY(dst, peer_copy(D, dst, RD.mem_rows.as<double>() + pos * d, s, RS.tmp.p,
                               8 * (size_t)k * d));
        GS_DTRY(dst, rank_sync(D, dst));
        pos += k;
      }
    }
    // every rank: clear the old index entries, fold its members (Eq. 3 in visit order)
    for (int r = 0; r < R; ++r) {
      gs_ctx* c = D->ctx[r];
      auto& RR = D->rk[r];
      GS_DCK(cudaSetDevice(D->dev[r]));
      cudaStream_t st = c->stream;
      const int64_t hl = nhl[r], m = m_r[r], hh = nhh[r];
      const int cmb = 1 - c->cur;
      if (m) {  // the combined list of the sweep (own + halos) still holds the index entries
        gs::k_idx_clear<<<blocks_for(hl + m + hh, 256), 256, 0, st>>>(
            (int)(hl + m + hh), c->ckey[cmb].as<uint32_t>(), c->idx.as<int32_t>());
        GS_DCK(cudaGetLastError());
      }
      const int64_t Mm = M[r];
      if (!Mm) {
        mnew[r] = 0;
        continue;
      }
      GS_DTRY(r, ensure_cells(c, Mm + 1, d));
      const unsigned mb = blocks_for(Mm, 256);
      std::vector<uint32_t> vseq(Mm);
      for (int64_t i = 0; i < Mm; ++i) vseq[i] = (uint32_t)i;
      GS_DCK(cudaMemcpyAsync(c->vals.p, vseq.data(), 4 * Mm, cudaMemcpyHostToDevice, st));
      const int kb = bits_for(box.vol_total);
      size_t tb = c->cub_tmp.bytes;
      GS_DCK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tb, RR.mem_key.as<uint32_t>(),
                                             c->skey.as<uint32_t>(), c->vals.as<uint32_t>(),
                                             c->sval.as<uint32_t>(), (int)Mm, 0, kb, st));
      gs::k_heads<<<mb, 256, 0, st>>>((int)Mm, c->skey.as<uint32_t>(), c->head.as<int32_t>());
      tb = c->cub_tmp.bytes;
      GS_DCK(cub::DeviceScan::InclusiveSum(c->cub_tmp.p, tb, c->head.as<int32_t>(),
                                           c->sid.as<int32_t>(), (int)Mm, st));
      gs::k_seg<<<mb, 256, 0, st>>>((int)Mm, c->head.as<int32_t>(), c->sid.as<int32_t>(),
                                    c->sval.as<uint32_t>(), c->parent.as<int32_t>(),
                                    c->segstart.as<int32_t>());
      GS_DCK(cudaGetLastError());
      int32_t mn = 0;
      GS_DCK(cudaMemcpyAsync(&mn, c->sid.as<int32_t>() + (Mm - 1), 4, cudaMemcpyDeviceToHost, st));
      GS_DCK(cudaStreamSynchronize(st));
      mnew[r] = mn;
      const int nxt = cmb;  // the combined buffer is free again
      switch (d) {
#define GS_CASE(DD)                                                                          \
  case DD:                                                                                   \
    gs::k_fold<DD><<<blocks_for(mn, 256), 256, 0, st>>>(                                     \
        mn, (int)Mm, c->segstart.as<int32_t>(), c->skey.as<uint32_t>(), c->sval.as<uint32_t>(), \
        RR.mem_cnt.as<uint32_t>(), RR.mem_rows.as<double>(), c->ckey[nxt].as<uint32_t>(),    \
        c->ccnt[nxt].as<uint32_t>(), c->S[nxt].as<double>());                                \
    break;
        GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
#undef GS_CASE
      }
      GS_DCK(cudaGetLastError());
      parent_local[r].resize(Mm);
      GS_DCK(cudaMemcpyAsync(parent_local[r].data(), c->parent.p, 4 * Mm, cudaMemcpyDeviceToHost,
                             st));
      gs::k_idx_set<<<blocks_for(mn, 256), 256, 0, st>>>(mn, c->ckey[nxt].as<uint32_t>(),
                                                        c->idx.as<int32_t>());
      GS_DCK(cudaGetLastError());
      GS_DCK(cudaStreamSynchronize(st));
      c->cur = nxt;
    }
    // the parent map in global ids, composed into the roots of the initial cells
    std::vector<int64_t> noff(R + 1, 0);
    for (int r = 0; r < R; ++r) noff[r + 1] = noff[r] + mnew[r];
    std::vector<int32_t> gparent(mt);
    for (int r = 0; r < R; ++r)
      for (int64_t j = 0; j < M[r]; ++j)
        gparent[mem_old[r][j]] = (int32_t)(noff[r] + parent_local[r][j]);
    for (int64_t i = 0; i < m0; ++i) root[i] = gparent[root[i]];
    // (4) has_converged over the new cells: the neighbours' new boundary layers in the index
    std::vector<std::vector<uint32_t>> nkey2(R);
    for (int r = 0; r < R; ++r) {
      gs_ctx* c = D->ctx[r];
      nkey2[r].resize(mnew[r]);
      GS_DCK(cudaSetDevice(D->dev[r]));
      if (mnew[r])
        GS_DCK(cudaMemcpy(nkey2[r].data(), c->ckey[c->cur].p, 4 * mnew[r], cudaMemcpyDeviceToHost));
    }
    int any_adj = 0;
    for (int r = 0; r < R; ++r) {
      gs_ctx* c = D->ctx[r];
      auto& RR = D->rk[r];
      if (!mnew[r]) continue;
      GS_DCK(cudaSetDevice(D->dev[r]));
      cudaStream_t st = c->stream;
      // boundary keys of the neighbours: r-1's last layer, r+1's first layer
      std::vector<uint32_t> bk;
      if (r > 0) {
        int64_t a, b;
        layer_ranges(box, nkey2[r - 1], lo[r - 1], hi[r - 1], &a, &b);
        bk.insert(bk.end(), nkey2[r - 1].begin() + b, nkey2[r - 1].end());
      }
      if (r + 1 < R) {
        int64_t a, b;
        layer_ranges(box, nkey2[r + 1], lo[r + 1], hi[r + 1], &a, &b);
        bk.insert(bk.end(), nkey2[r + 1].begin(), nkey2[r + 1].begin() + a);
      }
      const int64_t nb = (int64_t)bk.size();
      if (nb) {
        GS_DTRY(r, grow(c, RR.bkey, 4 * (size_t)nb));
        GS_DCK(cudaMemcpyAsync(RR.bkey.p, bk.data(), 4 * nb, cudaMemcpyHostToDevice, st));
        k_idx_mark<<<blocks_for(nb, 256), 256, 0, st>>>((int)nb, RR.bkey.as<uint32_t>(),
                                                        c->idx.as<int32_t>(), 1 << 30);
      }
      GS_DCK(cudaMemsetAsync(c->fadj.p, 0, 4, st));
      switch (d) {
#define GS_CASE(DD)                                                                        \
  case DD:                                                                                 \
    gs::k_adjacent<DD><<<blocks_for(mnew[r], 256), 256, 0, st>>>(                          \
        (int)mnew[r], box, K, c->ckey[c->cur].as<uint32_t>(), c->idx.as<int32_t>(),       \
        c->fdone.as<int32_t>(), c->fadj.as<int32_t>());                                    \
    break;
        GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6)
#undef GS_CASE
      }
      GS_DCK(cudaGetLastError());
      if (nb)
        k_idx_mark<<<blocks_for(nb, 256), 256, 0, st>>>((int)nb, RR.bkey.as<uint32_t>(),
                                                        c->idx.as<int32_t>(), -1);
      int32_t adj = 0;
      GS_DCK(cudaMemcpyAsync(&adj, c->fadj.p, 4, cudaMemcpyDeviceToHost, st));
      GS_DCK(cudaStreamSynchronize(st));
      any_adj |= adj;
    }
    for (int r = 0; r < R; ++r) {
      m_r[r] = mnew[r];
      off[r + 1] = off[r] + m_r[r];
    }
    D->hist_m.push_back(mt);
    D->hist_d.push_back(maxdisp);
    ++iter;
    conv = !any_adj || !any_changed;
    if (conv || iter >= cfg->max_iter) break;
  }
  // ---- 5. results: ids = global lex ranks; each rank labels its own points
  const int64_t k_all = off[R];
  D->d = d;
  D->nframes = 1;
  D->k.assign(1, k_all);
  D->cent.assign((size_t)k_all * d, 0.0);
  D->cent_off.assign(2, 0);
  D->cent_off[1] = k_all;
  for (int r = 0; r < R; ++r) {
    gs_ctx* c = D->ctx[r];
    if (!m_r[r]) continue;
    GS_DCK(cudaSetDevice(D->dev[r]));
    GS_DCK(cudaMemcpy(D->cent.data() + (size_t)off[r] * d, c->S[c->cur].p, 8 * m_r[r] * d,
                      cudaMemcpyDeviceToHost));
  }
  for (int r = 0; r < R; ++r) {
    gs_ctx* c = D->ctx[r];
    auto& RR = D->rk[r];
    GS_DCK(cudaSetDevice(D->dev[r]));
    cudaStream_t st = c->stream;
    // every rank's initial cells are in its index grid from the merge: clear them (clean
    // invariant), then the label table of ALL initial cells (any may hold this shard's points)
    if (m_r[r])
      gs::k_idx_clear<<<blocks_for(m_r[r], 256), 256, 0, st>>>(
          (int)m_r[r], c->ckey[c->cur].as<uint32_t>(), c->idx.as<int32_t>());
    GS_DTRY(r, grow(c, RR.mem_key, 4 * (size_t)m0));
    GS_DTRY(r, grow(c, RR.mem_idx, 4 * (size_t)m0));
    GS_DCK(cudaMemcpyAsync(RR.mem_key.p, init_key.data(), 4 * m0, cudaMemcpyHostToDevice, st));
    GS_DCK(cudaMemcpyAsync(RR.mem_idx.p, root.data(), 4 * m0, cudaMemcpyHostToDevice, st));
    k_lab_scatter<<<blocks_for(m0, 256), 256, 0, st>>>(m0, RR.mem_key.as<uint32_t>(),
                                                       RR.mem_idx.as<int32_t>(), c->lab.as<int32_t>());
    GS_DCK(cudaGetLastError());
    GS_DTRY(r, grow(c, c->labels, 4 * (size_t)pc[r]));
    gs::k_label<true><<<label_grid(c, pc[r], 1), 256, 0, st>>>(pc[r], 1, c->slot.p,
                                                          c->dbox.as<GsBox>(), c->lab.as<int32_t>(),
                                                          c->labels.as<int32_t>(), nullptr,
                                                          nullptr, 0, 0);
    GS_DCK(cudaGetLastError());
    GS_DCK(cudaMemcpyAsync(out->labels + p0[r], c->labels.p, 4 * pc[r], cudaMemcpyDeviceToHost, st));
    GS_DCK(cudaStreamSynchronize(st));
    c->shard_box = false;
    c->have_run = false;
  }
  out->k[0] = k_all;
  out->iterations[0] = iter;
  out->converged[0] = conv ? 1 : 0;
  if (!rec) {
    D->hist_m.clear();
    D->hist_d.clear();
  }
  D->have_run = true;
  return GS_OK;
}

}  // namespace

extern "C" {

gs_status gs_dist_create(int ndev, const int* devices, gs_dist** out) {
  if (!out || ndev < 1 || !devices) return GS_E_INVALID_PARAMETER;
  *out = nullptr;
  gs_dist* D = new gs_dist();
  D->R = ndev;
  D->dev.assign(devices, devices + ndev);
  D->rk.resize(ndev);
  for (int r = 0; r < ndev; ++r) {
    gs_ctx* c = nullptr;
    const gs_status s = gs_create(devices[r], nullptr, &c);
    if (s != GS_OK) {
      for (gs_ctx* x : D->ctx) gs_destroy(x);
      delete D;
      return s;
    }
    D->ctx.push_back(c);
  }
  // peer access between distinct devices (NVLink / NVSwitch); a refusal leaves the copies
  // staged by the driver, still correct
  for (int a = 0; a < ndev; ++a)
    for (int b = 0; b < ndev; ++b)
      if (devices[a] != devices[b]) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devices[a], devices[b]);
        if (can) {
          cudaSetDevice(devices[a]);
          cudaDeviceEnablePeerAccess(devices[b], 0);
          cudaGetLastError();
        }
      }
  *out = D;
  return GS_OK;
}

void gs_dist_destroy(gs_dist* D) {
  if (!D) return;
  for (int r = 0; r < D->R; ++r) {
    cudaSetDevice(D->dev[r]);
    for (DevBuf* b : {&D->rk[r].hh_key, &D->rk[r].hh_cnt, &D->rk[r].hh_rows, &D->rk[r].hl_key,
                      &D->rk[r].hl_cnt, &D->rk[r].hl_rows, &D->rk[r].out_rows, &D->rk[r].mem_idx,
                      &D->rk[r].mem_key, &D->rk[r].mem_cnt, &D->rk[r].mem_rows, &D->rk[r].nkey,
                      &D->rk[r].bkey, &D->rk[r].tmp})
      b->release();
    gs_destroy(D->ctx[r]);
  }
  delete D;
}

const char* gs_dist_last_error(const gs_dist* D) { return D ? D->err.c_str() : "null handle"; }

gs_status gs_dist_run_frames(gs_dist* D, const gs_input* in, const gs_config* cfg,
                             gs_result* out) {
  gs_status s = validate(in, cfg);
  if (s != GS_OK) return s;
  if (!D || !out || !out->labels || !out->k || !out->iterations || !out->converged)
    return GS_E_INVALID_PARAMETER;
  if (in->on_device) return dist_fail(D, GS_E_INVALID_PARAMETER, "frames are read from host memory");
  D->err.clear();
  D->have_run = false;
  const int R = D->R;
  const int64_t nf = in->batch, n = in->n;
  const size_t fb = input_bytes(in) / (size_t)nf;
  std::vector<int64_t> f0(R), fc(R);
  for (int r = 0; r < R; ++r) {
    const int64_t base = nf / R, rem = nf % R;
    f0[r] = r * base + std::min<int64_t>(r, rem);
    fc[r] = base + (r < rem ? 1 : 0);
  }
  std::vector<gs_status> st(R, GS_OK);
  std::vector<std::vector<double>> cent(R);
  std::vector<std::vector<int64_t>> coff(R);
  // one host thread per rank: each rank clusters its own frames, nothing crosses ranks
  std::vector<std::thread> th;
  for (int r = 0; r < R; ++r)
    th.emplace_back([&, r]() {
      if (!fc[r]) return;
      gs_input sub = *in;
      sub.points = static_cast<const char*>(in->points) + (size_t)f0[r] * fb;
      sub.batch = fc[r];
      gs_result res{out->labels + (size_t)f0[r] * n, out->k + f0[r], out->iterations + f0[r],
                    out->converged + f0[r]};
      st[r] = gs_run(D->ctx[r], &sub, cfg, &res);
      if (st[r] != GS_OK) return;
      for (int64_t f = 0; f < fc[r]; ++f) {
        coff[r].push_back((int64_t)cent[r].size() / in->d);
        std::vector<double> c((size_t)res.k[f] * in->d);
        st[r] = gs_get_centroids(D->ctx[r], f, c.data(), res.k[f]);
        if (st[r] != GS_OK) return;
        cent[r].insert(cent[r].end(), c.begin(), c.end());
      }
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < R; ++r)
    if (st[r] != GS_OK) return dist_fail(D, st[r], "rank " + std::to_string(r) + ": " + D->ctx[r]->err);
  D->d = in->d;
  D->nframes = nf;
  D->k.assign(out->k, out->k + nf);
  D->cent.clear();
  D->cent_off.assign(nf + 1, 0);
  for (int r = 0; r < R; ++r) {
    for (int64_t f = 0; f < fc[r]; ++f)
      D->cent_off[f0[r] + f] = (int64_t)D->cent.size() / in->d + coff[r][f];
    D->cent.insert(D->cent.end(), cent[r].begin(), cent[r].end());
  }
  D->cent_off[nf] = (int64_t)D->cent.size() / in->d;
  D->hist_m.clear();
  D->hist_d.clear();
  D->have_run = true;
  return GS_OK;
}

gs_status gs_dist_run_slabs(gs_dist* D, const gs_input* in, const gs_config* cfg,
                            gs_result* out) {
  gs_status s = validate(in, cfg);
  if (s != GS_OK) return s;
  if (!D || !out || !out->labels || !out->k || !out->iterations || !out->converged)
    return GS_E_INVALID_PARAMETER;
  D->err.clear();
  D->have_run = false;
  if (in->batch != 1) return dist_fail(D, GS_E_INVALID_PARAMETER, "slabs partition ONE cloud (batch 1)");
  if (in->d > 6) return dist_fail(D, GS_E_INVALID_PARAMETER, "slab sweeps: d <= 6");
  if (in->dtype == GS_U8 && in->d == 5)
    return dist_fail(D, GS_E_INVALID_PARAMETER, "rgbxy pixels cannot be sharded");
  if (in->on_device) return dist_fail(D, GS_E_INVALID_PARAMETER, "the cloud is read from host memory");
  s = slab_run(D, in, cfg, out);
  for (int r = 0; r < D->R; ++r) {  // a failed run leaves the ranks' grids to be rebuilt
    cudaSetDevice(D->dev[r]);
    cudaStreamSynchronize(D->ctx[r]->stream);
    D->ctx[r]->shard_box = false;
    D->ctx[r]->ctl_clean = false;
  }
  return s;
}

gs_status gs_dist_get_centroids(gs_dist* D, int64_t frame, double* out, int64_t cap_k) {
  if (!D || !out) return GS_E_INVALID_PARAMETER;
  if (!D->have_run || frame < 0 || frame >= D->nframes)
    return dist_fail(D, GS_E_INVALID_PARAMETER, "no such frame in the last run");
  const int64_t k = D->k[frame];
  if (cap_k < k) return dist_fail(D, GS_E_INVALID_PARAMETER, "centroid buffer too small");
  std::memcpy(out, D->cent.data() + (size_t)D->cent_off[frame] * D->d, sizeof(double) * k * D->d);
  return GS_OK;
}

gs_status gs_dist_get_history(gs_dist* D, int64_t* m_t, double* maxdisp_t, int32_t cap) {
  if (!D || !D->have_run) return GS_E_INVALID_PARAMETER;
  for (int32_t t = 0; t < cap && t < (int32_t)D->hist_m.size(); ++t) {
    if (m_t) m_t[t] = D->hist_m[t];
    if (maxdisp_t) maxdisp_t[t] = D->hist_d[t];
  }
  return GS_OK;
}

}  // extern "C"
