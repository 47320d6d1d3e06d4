// gs_oracle.cpp — CPU ORACLE for the GridShift hot path.  TEST INFRASTRUCTURE ONLY.
//
// This file is the parity checker, never the product: only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load liboracle.  The product
// path (libgridshift_cuda.so) has no CPU fallback and never links this file.
//
// It restates, line by line, the reference specification of the path:
//   grid-core  /root/reference/SPEC.md:17-100   (grid_index, neighborhood,
//              build_active_grid, merge_into, invariants :77-81, ledger :83-87)
//   engine     /root/reference/SPEC.md:102-181  (iterate_once :117-125, has_converged
//              :126-134, run :135-143, ledger :161-167)
//   Alg. 1     /root/reference/PAPER.md:83-118 read through SPEC's typo fixes SPEC.md:163-164,
//              Eq. (3)-(5) PAPER.md:68-78, :124-130.
// The reference ships no implementation code, so there is no `oracle/_ref`:
// this restatement is pinned against every known-answer example the SPEC holds
// (tests/golden/spec_kats.json, tests/test_oracle_kat.py).
//
// Pins the SPEC leaves open (DESIGN.md §"Oracle pins"):
//   P1 grid_index is floor(RN(x/h)) with IEEE division, never x*(1/h)
//   P2 sweep sum: num = 0.0; for v in lex order: num = num + (double)C'*S'; S = num/(double)ΣC'
//      (no FMA: build with -ffp-contract=off)                                  SPEC.md:120(c), :52
//   P3 a cell with no active neighbour other than itself keeps its centroid bit-for-bit
//                                                                              SPEC.md:124
//   P4 merge (Eq. 3) folded in visit order: s = ((double)c*s + (double)C'*S') / (double)(c+C')
//                                                                              SPEC.md:70, :75
//   P5 do-while loop: >= 1 iteration; exit on has_converged || !changed || iters == max_iter
//                                                                              SPEC.md:138, :141, :164
//   P6 build mode 0 ("spec"): incremental mean in point order (Alg. 1 line 5).
//      build mode 1 ("fixed"): the GPU engine's deterministic fixed-point cell sums
//      (DESIGN.md §"Fixed-point binning"); every later step is identical in both modes.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <vector>

namespace {

constexpr int kMaxD = 12;  // SPEC.md:96 documented limit d <= 12

// Status codes shared with include/gridshift_c.h (gs_status).
enum {
  OK = 0,
  E_INVALID_INPUT = 1,
  E_INVALID_BANDWIDTH = 2,
  E_EMPTY_INPUT = 3,
  E_INVALID_PARAMETER = 4,
  E_INTERNAL_INVARIANT = 5,
  E_TUNING_FAILED = 11,
  E_UNDEFINED_SCORE = 12,
  E_INVALID_WINDOW = 13,
  E_SELECTION = 14,
};

using Key = std::array<int64_t, kMaxD>;  // GridIndex; unused tail is zero

struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t h = 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < kMaxD; ++i) {
      h ^= (uint64_t)k[i] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    }
    return (size_t)h;
  }
};

// CellRecord: centroid, count, member set.
struct Cell {
  Key key;
  double c[kMaxD];
  int64_t count;
  std::vector<int64_t> members;
};

// grid_index: floor toward -inf of the IEEE quotient (pin P1).
inline int64_t grid_coord(double x, double h) { return (int64_t)std::floor(x / h); }

// Fixed-point scale exponent for build mode 1: |sum of offsets * 2^F| < 2^61 for any cell
// of at most n points (offsets lie in [~0, h]).  Mirrors gs_fixed_shift() in the CUDA engine.
int fixed_shift(int64_t n, double h) {
  int ln = 0;
  while ((int64_t(1) << ln) < n) ++ln;            // ceil(log2(n))
  int eh = std::ilogb(h) + 1;                      // h < 2^eh
  int F = 61 - ln - eh;
  if (F > 1000) F = 1000;
  if (F < -1000) F = -1000;
  return F;
}

struct Engine {
  int d;
  double h;
  std::vector<Cell> cells;  // kept sorted lexicographically by key between iterations

  // neighborhood: the 3^d offsets in lexicographic order of v.
  static std::vector<std::array<int8_t, kMaxD>> offsets(int d) {
    std::vector<std::array<int8_t, kMaxD>> out;
    int64_t total = 1;
    for (int i = 0; i < d; ++i) total *= 3;
    for (int64_t t = 0; t < total; ++t) {
      std::array<int8_t, kMaxD> v{};
      int64_t r = t;
      for (int i = d - 1; i >= 0; --i) {  // dim 0 is the most significant digit
        v[i] = (int8_t)(r % 3) - 1;
        r /= 3;
      }
      out.push_back(v);
    }
    return out;
  }

  void sort_cells() {
    std::sort(cells.begin(), cells.end(),
              [](const Cell& a, const Cell& b) { return a.key < b.key; });
  }

  // build_active_grid.
  int build(const double* X, int64_t n, int mode, int64_t* slot_out) {
    std::unordered_map<Key, int64_t, KeyHash> index;
    index.reserve((size_t)std::min<int64_t>(n, 1 << 22));
    std::vector<int64_t> cell_of(n);
    int F = fixed_shift(n, h);
    double scale = std::ldexp(1.0, F);
    std::vector<std::array<int64_t, kMaxD>> qsum;
    for (int64_t i = 0; i < n; ++i) {
      Key k{};
      const double* x = X + i * d;
      for (int c = 0; c < d; ++c) {
        if (!std::isfinite(x[c])) return E_INVALID_INPUT;
        k[c] = grid_coord(x[c], h);
      }
      auto it = index.find(k);
      int64_t ci;
      if (it == index.end()) {
        ci = (int64_t)cells.size();
        index.emplace(k, ci);
        Cell cell;
        cell.key = k;
        for (int c = 0; c < d; ++c) cell.c[c] = x[c];  // Alg. 1 lines 8-10
        cell.count = 1;
        cells.push_back(std::move(cell));
        qsum.push_back({});
      } else {
        ci = it->second;
        Cell& cell = cells[ci];
        for (int c = 0; c < d; ++c)  // Alg. 1 line 5: S <- (C*S + x)/(C+1)
          cell.c[c] = ((double)cell.count * cell.c[c] + x[c]) / (double)(cell.count + 1);
        cell.count += 1;
      }
      cells[ci].members.push_back(i);
      cell_of[i] = ci;
      if (mode == 1) {
        for (int c = 0; c < d; ++c) {
          double base = (double)k[c] * h;
          double off = x[c] - base;
          qsum[ci][c] += (int64_t)std::nearbyint(off * scale);
        }
      }
    }
    if (mode == 1) {
      for (size_t ci = 0; ci < cells.size(); ++ci) {
        Cell& cell = cells[ci];
        for (int c = 0; c < d; ++c) {
          double base = (double)cell.key[c] * h;
          double mean_q = (double)qsum[ci][c] / (double)cell.count;
          cell.c[c] = base + std::ldexp(mean_q, -F);
        }
      }
    }
    // Lex order, and remember each point's initial cell rank (slot) for the GPU K2 check.
    std::vector<int64_t> perm(cells.size());
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = (int64_t)i;
    std::sort(perm.begin(), perm.end(),
              [&](int64_t a, int64_t b) { return cells[a].key < cells[b].key; });
    std::vector<int64_t> rank(cells.size());
    for (size_t r = 0; r < perm.size(); ++r) rank[perm[r]] = (int64_t)r;
    if (slot_out)
      for (int64_t i = 0; i < n; ++i) slot_out[i] = rank[cell_of[i]];
    sort_cells();
    return OK;
  }

  // lookup of an OLD key among the lex-sorted snapshot (binary search; -1 if inactive).
  int64_t find(const std::vector<Key>& keys, const Key& k) const {
    auto it = std::lower_bound(keys.begin(), keys.end(), k);
    if (it == keys.end() || *it != k) return -1;
    return (int64_t)(it - keys.begin());
  }

  // iterate_once.  parent[i] = rank of the new cell that old cell i joined.
  int iterate_once(bool* changed, double* maxdisp, std::vector<int64_t>* parent,
                   std::vector<double>* swept) {
    const int64_t m = (int64_t)cells.size();
    const auto offs = offsets(d);
    // (a) snapshot: C' counts and S' centroids (S' is then updated in place, Eq. 5)
    std::vector<Key> keys(m);
    std::vector<int64_t> Cs(m);
    std::vector<double> S((size_t)m * d), S0((size_t)m * d);
    for (int64_t i = 0; i < m; ++i) {
      keys[i] = cells[i].key;
      Cs[i] = cells[i].count;
      for (int c = 0; c < d; ++c) S[i * d + c] = S0[i * d + c] = cells[i].c[c];
    }
    // (b)+(c) lexicographic in-place sweep
    for (int64_t i = 0; i < m; ++i) {
      double num[kMaxD];
      for (int c = 0; c < d; ++c) num[c] = 0.0;
      int64_t den = 0;
      int others = 0;
      for (size_t t = 0; t < offs.size(); ++t) {
        Key k = keys[i];
        bool self = true;
        for (int c = 0; c < d; ++c) {
          k[c] += offs[t][c];
          if (offs[t][c] != 0) self = false;
        }
        int64_t nb = self ? i : find(keys, k);
        if (nb < 0) continue;
        double w = (double)Cs[nb];
        for (int c = 0; c < d; ++c) num[c] = num[c] + w * S[nb * d + c];
        den += Cs[nb];
        if (!self) ++others;
      }
      if (others == 0) continue;  // pin P3
      for (int c = 0; c < d; ++c) S[i * d + c] = num[c] / (double)den;
    }
    if (swept) *swept = S;
    // displacement history and (e) changed
    bool ch = false;
    double md = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int c = 0; c < d; ++c) {
        double t = S[i * d + c] - S0[i * d + c];
        acc = acc + t * t;
        if (std::memcmp(&S[i * d + c], &S0[i * d + c], sizeof(double)) != 0) ch = true;
      }
      double disp = std::sqrt(acc);
      if (disp > md) md = disp;
    }
    // (d) rehome each cell, in visit order, via merge_into (Eq. 3-4)
    std::unordered_map<Key, int64_t, KeyHash> nidx;
    std::vector<Cell> next;
    std::vector<int64_t> par(m);
    for (int64_t i = 0; i < m; ++i) {
      Key k{};
      for (int c = 0; c < d; ++c) k[c] = grid_coord(S[i * d + c], h);
      if (k != keys[i]) ch = true;
      auto it = nidx.find(k);
      if (it == nidx.end()) {  // key absent -> inserted as-is
        Cell cell;
        cell.key = k;
        for (int c = 0; c < d; ++c) cell.c[c] = S[i * d + c];
        cell.count = Cs[i];
        cell.members = std::move(cells[i].members);
        par[i] = (int64_t)next.size();
        nidx.emplace(k, par[i]);
        next.push_back(std::move(cell));
      } else {  // Eq. (3): count-weighted mean, counts add, member sets union
        Cell& cell = next[it->second];
        for (int c = 0; c < d; ++c)
          cell.c[c] = ((double)cell.count * cell.c[c] + (double)Cs[i] * S[i * d + c]) /
                      (double)(cell.count + Cs[i]);
        cell.count += Cs[i];
        cell.members.insert(cell.members.end(), cells[i].members.begin(),
                            cells[i].members.end());
        par[i] = it->second;
      }
    }
    // re-rank new cells lexicographically
    std::vector<int64_t> perm(next.size());
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = (int64_t)i;
    std::sort(perm.begin(), perm.end(),
              [&](int64_t a, int64_t b) { return next[a].key < next[b].key; });
    std::vector<int64_t> rank(next.size());
    for (size_t r = 0; r < perm.size(); ++r) rank[perm[r]] = (int64_t)r;
    for (int64_t i = 0; i < m; ++i) par[i] = rank[par[i]];
    std::vector<Cell> sorted;
    sorted.reserve(next.size());
    for (size_t r = 0; r < perm.size(); ++r) sorted.push_back(std::move(next[perm[r]]));
    cells = std::move(sorted);
    if ((int64_t)cells.size() > m) return E_INTERNAL_INVARIANT;  // (f) |map'| <= |map|
    if (parent) *parent = std::move(par);
    *changed = ch;
    *maxdisp = md;
    return OK;
  }

  // has_converged: no active cell has another active cell in its 1-neighborhood.
  bool has_converged() const {
    const int64_t m = (int64_t)cells.size();
    std::vector<Key> keys(m);
    for (int64_t i = 0; i < m; ++i) keys[i] = cells[i].key;
    const auto offs = offsets(d);
    for (int64_t i = 0; i < m; ++i) {
      for (const auto& v : offs) {
        Key k = keys[i];
        bool self = true;
        for (int c = 0; c < d; ++c) {
          k[c] += v[c];
          if (v[c] != 0) self = false;
        }
        if (!self && find(keys, k) >= 0) return false;
      }
    }
    return true;
  }
};

int check_common(int64_t n, int d, double h) {
  if (!(h > 0.0) || !std::isfinite(h)) return E_INVALID_BANDWIDTH;
  if (n < 1) return E_EMPTY_INPUT;
  if (d < 1 || d > kMaxD) return E_INVALID_PARAMETER;
  return OK;
}

}  // namespace

extern "C" {

int gso_version() { return 1; }

int gso_fixed_shift(int64_t n, double h) { return fixed_shift(n, h); }

// build_active_grid only: returns m0 and the lex-sorted cells; slot[i] = rank of point i's cell.
// keys_out: m0*d int64; counts_out: m0; cent_out: m0*d; caller sizes them for n cells.
int gso_build(const double* X, int64_t n, int32_t d, double h, int32_t mode, int64_t* m_out,
              int64_t* keys_out, int64_t* counts_out, double* cent_out, int64_t* slot_out) {
  int st = check_common(n, d, h);
  if (st) return st;
  Engine e{d, h, {}};
  st = e.build(X, n, mode, slot_out);
  if (st) return st;
  *m_out = (int64_t)e.cells.size();
  for (size_t i = 0; i < e.cells.size(); ++i) {
    for (int c = 0; c < d; ++c) {
      keys_out[i * d + c] = e.cells[i].key[c];
      cent_out[i * d + c] = e.cells[i].c[c];
    }
    counts_out[i] = e.cells[i].count;
  }
  return OK;
}

// One iterate_once on an injected state (lex-sorted keys).  Outputs the new state, the
// post-sweep centroids (pre-merge), parent ranks, changed and has_converged(new state).
int gso_iterate_once(int32_t d, double h, int64_t m, const int64_t* keys, const int64_t* counts,
                     const double* cent, int64_t* m_out, int64_t* keys_out,
                     int64_t* counts_out, double* cent_out, double* swept_out,
                     int64_t* parent_out, int32_t* changed_out, int32_t* converged_out,
                     double* maxdisp_out) {
  int st = check_common(m, d, h);
  if (st) return st;
  Engine e{d, h, {}};
  e.cells.resize(m);
  for (int64_t i = 0; i < m; ++i) {
    Key k{};
    for (int c = 0; c < d; ++c) {
      k[c] = keys[i * d + c];
      e.cells[i].c[c] = cent[i * d + c];
    }
    e.cells[i].key = k;
    e.cells[i].count = counts[i];
    e.cells[i].members = {i};
    if (counts[i] < 1) return E_INVALID_INPUT;
    if (i > 0 && !(e.cells[i - 1].key < k)) return E_INVALID_INPUT;  // must be strictly lex-sorted
  }
  bool changed;
  double md;
  std::vector<int64_t> parent;
  std::vector<double> swept;
  st = e.iterate_once(&changed, &md, &parent, &swept);
  if (st) return st;
  *m_out = (int64_t)e.cells.size();
  for (size_t i = 0; i < e.cells.size(); ++i) {
    for (int c = 0; c < d; ++c) {
      keys_out[i * d + c] = e.cells[i].key[c];
      cent_out[i * d + c] = e.cells[i].c[c];
    }
    counts_out[i] = e.cells[i].count;
  }
  for (int64_t i = 0; i < m; ++i) parent_out[i] = parent[i];
  std::memcpy(swept_out, swept.data(), sizeof(double) * (size_t)m * d);
  *changed_out = changed ? 1 : 0;
  *converged_out = e.has_converged() ? 1 : 0;
  *maxdisp_out = md;
  return OK;
}

// has_converged on a given key set (lex order not required).
int gso_has_converged(int32_t d, int64_t m, const int64_t* keys, int32_t* out) {
  Engine e{d, 1.0, {}};
  e.cells.resize(m);
  for (int64_t i = 0; i < m; ++i) {
    Key k{};
    for (int c = 0; c < d; ++c) k[c] = keys[i * d + c];
    e.cells[i].key = k;
  }
  e.sort_cells();
  *out = e.has_converged() ? 1 : 0;
  return OK;
}

// engine.run on one dataset (one frame).
//   labels_out: n int32 cluster ids (lex rank of the final cell)
//   cent_out:   capacity n*d; first k*d entries are the cluster centroids in id order
//   hist_m / hist_disp: capacity max_iter; per-iteration active-cell count entering the
//   iteration and max sweep displacement; *iters_out entries are written.
int gso_run(const double* X, int64_t n, int32_t d, double h, int32_t max_iter, int32_t mode,
            int32_t* labels_out, int64_t* k_out, int32_t* iters_out, int32_t* converged_out,
            double* cent_out, int64_t* hist_m, double* hist_disp) {
  int st = check_common(n, d, h);
  if (st) return st;
  if (max_iter < 1) return E_INVALID_PARAMETER;  // SPEC.md:112 positive integer
  Engine e{d, h, {}};
  st = e.build(X, n, mode, nullptr);
  if (st) return st;
  int iters = 0;
  bool conv = false;
  do {  // pin P5: do-while
    int64_t m_t = (int64_t)e.cells.size();
    bool changed;
    double md;
    st = e.iterate_once(&changed, &md, nullptr, nullptr);
    if (st) return st;
    if (hist_m) hist_m[iters] = m_t;
    if (hist_disp) hist_disp[iters] = md;
    ++iters;
    if (e.has_converged() || !changed) {
      conv = true;
      break;
    }
  } while (iters < max_iter);
  // ClusterLabeling: ids by lexicographic order of final keys (cells are kept sorted)
  int64_t seen = 0;
  for (size_t id = 0; id < e.cells.size(); ++id) {
    for (int64_t p : e.cells[id].members) {
      if (p < 0 || p >= n) return E_INTERNAL_INVARIANT;
      labels_out[p] = (int32_t)id;
      ++seen;
    }
    for (int c = 0; c < d; ++c) cent_out[id * d + c] = e.cells[id].c[c];
  }
  if (seen != n) return E_INTERNAL_INVARIANT;  // partition invariant SPEC.md:78
  *k_out = (int64_t)e.cells.size();
  *iters_out = iters;
  *converged_out = conv ? 1 : 0;
  return OK;
}

}  // extern "C"

// ---- metrics: silhouette_subsampled + tune_bandwidth (ledger :342-348) ----
// Pins the SPEC leaves open (DESIGN.md §"Bandwidth sweep"):
//   S1 subsample ("seeded uniform subsample of min(n, cap) points"): n <= cap
//      takes every point; else a partial Fisher-Yates over [0, n) driven by SplitMix64(seed)
//      (j = i + next() % (n - i), swap), the first cap positions, sorted ascending;
//   S2 silhouette: dist = sqrt(sum_c (xi_c - xj_c)^2), terms in c order, no
//      FMA; for point i the clusters of the sample are walked in ascending label order and
//      their members in ascending sample position, each cluster's distances summed in that
//      order (i itself skipped); a = sum/(size-1) over i's own cluster, b = min over the others
//      of sum/size; s_i = (b - a)/max(a, b), 0 when i's cluster is a singleton or max(a,b)==0;
//      score = (sum of s_i in sample order) / s;
//   S3 a sweep entry is undefined when the sample holds < 2 clusters;
//      best_h = max score, ties -> smallest h (first in grid order after sorting by h).
namespace {
uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double sq_dist(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int c = 0; c < d; ++c) {
    const double t = a[c] - b[c];
    acc = acc + t * t;
  }
  return std::sqrt(acc);
}
}  // namespace

extern "C" {

int64_t gso_sample_indices(int64_t n, int64_t cap, uint64_t seed, int64_t* out) {
  if (n <= cap) {
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    return n;
  }
  std::unordered_map<int64_t, int64_t> sw;  // sparse Fisher-Yates: only touched slots
  auto at = [&](int64_t i) {
    auto it = sw.find(i);
    return it == sw.end() ? i : it->second;
  };
  uint64_t st = seed;
  for (int64_t i = 0; i < cap; ++i) {
    const int64_t j = i + (int64_t)(splitmix64(st) % (uint64_t)(n - i));
    const int64_t vi = at(i), vj = at(j);
    sw[i] = vj;
    sw[j] = vi;
    out[i] = vj;
  }
  std::sort(out, out + cap);
  return cap;
}

// silhouette (pin S2) of s points (row-major s x d) with labels.
// Returns E_INVALID_PARAMETER-free status; *valid = 0 when fewer than 2 clusters.
int gso_silhouette(const double* X, const int32_t* labels, int64_t s, int32_t d, double* score,
                   int32_t* valid, double* per_point) {
  std::vector<int64_t> ord(s);
  for (int64_t i = 0; i < s; ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(),
                   [&](int64_t a, int64_t b) { return labels[a] < labels[b]; });
  std::vector<int64_t> seg;  // cluster starts in ord
  for (int64_t t = 0; t < s; ++t)
    if (t == 0 || labels[ord[t]] != labels[ord[t - 1]]) seg.push_back(t);
  const int64_t kc = (int64_t)seg.size();
  seg.push_back(s);
  *valid = kc >= 2 ? 1 : 0;
  *score = 0.0;
  if (kc < 2) return OK;
  double total = 0.0;
  for (int64_t i = 0; i < s; ++i) {
    double a = 0.0, b = INFINITY;
    bool single = false;
    for (int64_t c = 0; c < kc; ++c) {
      double sum = 0.0;
      for (int64_t t = seg[c]; t < seg[c + 1]; ++t) {
        const int64_t j = ord[t];
        if (j == i) continue;
        sum = sum + sq_dist(X + i * d, X + j * d, d);
      }
      const int64_t size = seg[c + 1] - seg[c];
      if (labels[ord[seg[c]]] == labels[i]) {
        if (size == 1) single = true;
        else a = sum / (double)(size - 1);
      } else {
        const double mean = sum / (double)size;
        if (mean < b) b = mean;
      }
    }
    const double mx = a > b ? a : b;
    const double si = (single || mx == 0.0) ? 0.0 : (b - a) / mx;
    if (per_point) per_point[i] = si;
    total = total + si;
  }
  *score = total / (double)s;
  return OK;
}

// tune_bandwidth with silhouette_subsampled: per h the
// engine run (build `mode`), its cluster count and iterations, the subsample silhouette.
int gso_tune(const double* X, int64_t n, int32_t d, const double* hs, int32_t nh,
             int32_t max_iter, int64_t cap, uint64_t seed, int32_t mode, double* scores,
             int64_t* ks, int32_t* iters, int32_t* valid, double* best_h) {
  if (nh < 1 || cap < 2) return E_INVALID_PARAMETER;
  for (int32_t i = 0; i < nh; ++i)
    if (!(hs[i] > 0.0 && hs[i] <= 1.0)) return E_INVALID_BANDWIDTH;
  std::vector<int64_t> idx((size_t)std::min(n, cap));
  const int64_t s = gso_sample_indices(n, cap, seed, idx.data());
  std::vector<double> xs((size_t)(s * d));
  for (int64_t t = 0; t < s; ++t)
    for (int c = 0; c < d; ++c) xs[t * d + c] = X[idx[t] * d + c];
  std::vector<int32_t> lab(n), ls(s);
  std::vector<double> cent((size_t)(n * d));
  int best = -1;
  for (int32_t i = 0; i < nh; ++i) {
    int32_t conv;
    int st = gso_run(X, n, d, hs[i], max_iter, mode, lab.data(), &ks[i], &iters[i], &conv,
                     cent.data(), nullptr, nullptr);
    if (st) return st;
    for (int64_t t = 0; t < s; ++t) ls[t] = lab[idx[t]];
    gso_silhouette(xs.data(), ls.data(), s, d, &scores[i], &valid[i], nullptr);
    if (valid[i] && (best < 0 || scores[i] > scores[best] ||
                     (scores[i] == scores[best] && hs[i] < hs[best])))
      best = i;
  }
  if (best < 0) return E_TUNING_FAILED;
  *best_h = hs[best];
  return OK;
}

}  // extern "C"

// ---- tracker: GridShift object tracking, Algorithm 2 ----
// Pins the SPEC leaves open (DESIGN.md §"Tracker"):
//   T1 window W(o, l, w) = pixels (x, y) with ceil(ox - l*0.5) <= x <= floor(ox + l*0.5) and
//      ceil(oy - w*0.5) <= y <= floor(oy + w*0.5), clipped to the frame;
//   T2 colour cell of a pixel: k_c = floor((v_c / 255.0) / h) per channel (the segmentation
//      features, and grid_index); id (k_r*K + k_g)*K + k_b, K = floor(1/h)+1;
//   T3 init: engine.run on the window's (r,g,b)/255 in row-major pixel order;
//      top_k = the k largest clusters by pixel count (ties -> smaller id) or explicit ids;
//      B = colour cells of the selected pixels;
//   T4 track_frame: per inner iteration: region W(o, l/f, w/f); R = region
//      pixels whose cell is in B; R empty -> l, w *= 1.1; else o' = (sum x / |R|, sum y / |R|),
//      B = cells of R, l *= (max x - min x < l) ? 0.99 : 1.01 (w likewise on y), and the loop
//      ends when sqrt(dx*dx + dy*dy) < eta; at most max_inner iterations; lost = R was empty
//      in every iteration;
//   T5 track_sequence: frames[0] initialises, frames 1..T-1 are tracked.
namespace {
struct TrackState {
  double ox, oy, l, w;
  std::vector<uint8_t> B;  // K^3 cell bitmap (one byte per cell here)
};

int track_cells(double h, int* K_out) {
  const double K = std::floor(1.0 / h) + 1.0;
  if (!(K >= 1.0) || K * K * K > (double)(1 << 22)) return E_INVALID_PARAMETER;
  *K_out = (int)K;
  return OK;
}

inline int pixel_cell(const uint8_t* px, double h, int K) {
  int id = 0;
  for (int c = 0; c < 3; ++c) id = id * K + (int)std::floor(((double)px[c] / 255.0) / h);
  return id;
}

bool window_range(double o, double len, int lim, int* lo, int* hi) {
  const double a = std::ceil(o - len * 0.5), b = std::floor(o + len * 0.5);
  const double ca = std::max(a, 0.0), cb = std::min(b, (double)(lim - 1));
  if (!(ca <= cb)) return false;
  *lo = (int)ca;
  *hi = (int)cb;
  return true;
}
}  // namespace

extern "C" {

int gso_track(const uint8_t* frames, int64_t T, int32_t H, int32_t W, const double* win0,
              double h, double f, double eta, int32_t max_inner, int32_t engine_max_iter,
              int32_t top_k, const int32_t* ids, int32_t n_ids, int32_t mode, double* out_win,
              int32_t* out_lost, int32_t* out_inner) {
  if (!(h > 0.0) || !std::isfinite(h)) return E_INVALID_BANDWIDTH;
  if (T < 1 || H < 1 || W < 1 || !(f >= 1.0) || !(eta > 0.0) || max_inner < 1 ||
      engine_max_iter < 1 || (n_ids == 0 && top_k < 1) || !(win0[2] > 0.0) || !(win0[3] > 0.0))
    return E_INVALID_PARAMETER;
  int K;
  if (track_cells(h, &K)) return E_INVALID_PARAMETER;
  const int64_t fpx = (int64_t)H * W;
  // ---- T3: init on frames[0]
  int x0, x1, y0, y1;
  if (!window_range(win0[0], win0[2], W, &x0, &x1) || !window_range(win0[1], win0[3], H, &y0, &y1))
    return E_INVALID_WINDOW;
  const int cw = x1 - x0 + 1, ch = y1 - y0 + 1;
  const int64_t np = (int64_t)cw * ch;
  std::vector<double> X((size_t)(np * 3));
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x) {
      const uint8_t* px = frames + ((int64_t)y * W + x) * 3;
      const int64_t q = (int64_t)(y - y0) * cw + (x - x0);
      for (int c = 0; c < 3; ++c) X[q * 3 + c] = (double)px[c] / 255.0;
    }
  std::vector<int32_t> lab(np);
  std::vector<double> cent((size_t)(np * 3));
  int64_t k;
  int32_t it, cv;
  int st = gso_run(X.data(), np, 3, h, engine_max_iter, mode, lab.data(), &k, &it, &cv,
                   cent.data(), nullptr, nullptr);
  if (st) return st;
  std::vector<int64_t> size(k, 0);
  for (int64_t q = 0; q < np; ++q) ++size[lab[q]];
  std::vector<uint8_t> sel(k, 0);
  if (n_ids > 0) {
    for (int32_t i = 0; i < n_ids; ++i) {
      if (ids[i] < 0 || ids[i] >= k) return E_SELECTION;
      sel[ids[i]] = 1;
    }
  } else {
    std::vector<int64_t> ord(k);
    for (int64_t c = 0; c < k; ++c) ord[c] = c;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return size[a] > size[b]; });
    for (int64_t r = 0; r < std::min<int64_t>(top_k, k); ++r) sel[ord[r]] = 1;
  }
  TrackState s{win0[0], win0[1], win0[2], win0[3], std::vector<uint8_t>((size_t)K * K * K, 0)};
  for (int y = y0; y <= y1; ++y)
    for (int x = x0; x <= x1; ++x)
      if (sel[lab[(int64_t)(y - y0) * cw + (x - x0)]])
        s.B[pixel_cell(frames + ((int64_t)y * W + x) * 3, h, K)] = 1;
  // ---- T4/T5
  std::vector<uint8_t> nb(s.B.size());
  for (int64_t t = 1; t < T; ++t) {
    const uint8_t* fr = frames + t * fpx * 3;
    bool found = false;
    int inner = 0;
    for (int itn = 0; itn < max_inner; ++itn) {
      ++inner;
      int64_t cnt = 0, sx = 0, sy = 0;
      int mnx = W, mxx = -1, mny = H, mxy = -1;
      std::fill(nb.begin(), nb.end(), 0);
      int a0, a1, b0, b1;
      const double lr = s.l / f, wr = s.w / f;
      if (window_range(s.ox, lr, W, &a0, &a1) && window_range(s.oy, wr, H, &b0, &b1)) {
        for (int y = b0; y <= b1; ++y)
          for (int x = a0; x <= a1; ++x) {
            const int cell = pixel_cell(fr + ((int64_t)y * W + x) * 3, h, K);
            if (!s.B[cell]) continue;
            ++cnt;
            sx += x;
            sy += y;
            mnx = std::min(mnx, x);
            mxx = std::max(mxx, x);
            mny = std::min(mny, y);
            mxy = std::max(mxy, y);
            nb[cell] = 1;
          }
      }
      if (cnt == 0) {  // target lost in this region: grow the window (Alg. 2 lines 9-10)
        s.l = s.l * 1.1;
        s.w = s.w * 1.1;
        continue;
      }
      found = true;
      const double nx = (double)sx / (double)cnt, ny = (double)sy / (double)cnt;
      s.B.swap(nb);
      s.l = ((double)(mxx - mnx) < s.l) ? s.l * 0.99 : s.l * 1.01;
      s.w = ((double)(mxy - mny) < s.w) ? s.w * 0.99 : s.w * 1.01;
      const double dx = nx - s.ox, dy = ny - s.oy;
      const double disp = std::sqrt(dx * dx + dy * dy);
      s.ox = nx;
      s.oy = ny;
      if (disp < eta) break;
    }
    double* o = out_win + (t - 1) * 4;
    o[0] = s.ox;
    o[1] = s.oy;
    o[2] = s.l;
    o[3] = s.w;
    out_lost[t - 1] = found ? 0 : 1;
    out_inner[t - 1] = inner;
  }
  return OK;
}

}  // extern "C"

// ---- baselines: MS++ per-point grid mean shift, parallel (Jacobi) updates ----
// Pins the SPEC leaves open (DESIGN.md §"MS++"):
//   M1 cell centroids are the fixed-point means of build mode 1 (F = fixed_shift(n, h)), for the
//      first grid over the points and every re-grid over the moved particles (a particle of
//      count c adds c*q);
//   M2 update (Eq. 6): every cell j at once from the previous state:
//      num = 0.0; num = num + (double)C(j+v)*S(j+v) over active neighbours in lex v order;
//      S'(j) = num / (double)sum C; a cell with no active neighbour but itself keeps S (P3);
//   M3 every point / particle of cell j moves to S'(j); the iteration's displacement is the max
//      over points (first iteration) or particles of sqrt(sum_c (S'_c - x_c)^2);
//   M4 particles that share a cell coincide after the move and merge (counts add); the loop is a
//      do-while: stop when displacement < tol or after max_iter iterations;
//   M5 final clusters: the cells of the final particles, ids by lex key order,
//      centroids their fixed-point means.
namespace {
struct MsCells {
  std::vector<Key> key;
  std::vector<int64_t> cnt;
  std::vector<double> S;  // m x d
};

// re-grid particles (pos m_p x d, counts) into lex-sorted cells; cell_of[i] = cell rank
void ms_regrid(const std::vector<double>& pos, const std::vector<int64_t>& pc, int d, double h,
               int F, MsCells* out, std::vector<int64_t>* cell_of) {
  const int64_t mp = (int64_t)pc.size();
  const double scale = std::ldexp(1.0, F);
  std::vector<std::pair<Key, int64_t>> kp(mp);
  for (int64_t i = 0; i < mp; ++i) {
    Key k{};
    for (int c = 0; c < d; ++c) k[c] = grid_coord(pos[i * d + c], h);
    kp[i] = {k, i};
  }
  std::sort(kp.begin(), kp.end());
  out->key.clear();
  out->cnt.clear();
  out->S.clear();
  cell_of->assign(mp, -1);
  std::vector<int64_t> qs;
  for (int64_t t = 0; t < mp; ++t) {
    const Key& k = kp[t].first;
    const int64_t i = kp[t].second;
    if (t == 0 || !(kp[t - 1].first == k)) {
      out->key.push_back(k);
      out->cnt.push_back(0);
      qs.resize(qs.size() + d, 0);
    }
    const int64_t r = (int64_t)out->key.size() - 1;
    (*cell_of)[i] = r;
    out->cnt[r] += pc[i];
    for (int c = 0; c < d; ++c) {
      const double off = pos[i * d + c] - (double)k[c] * h;
      qs[r * d + c] += pc[i] * (int64_t)std::nearbyint(off * scale);
    }
  }
  const int64_t m = (int64_t)out->key.size();
  out->S.resize(m * d);
  for (int64_t r = 0; r < m; ++r)
    for (int c = 0; c < d; ++c)
      out->S[r * d + c] = (double)out->key[r][c] * h +
                          std::ldexp((double)qs[r * d + c] / (double)out->cnt[r], -F);
}

void ms_jacobi(const MsCells& g, int d, std::vector<double>* Snew) {
  const int64_t m = (int64_t)g.cnt.size();
  std::unordered_map<Key, int64_t, KeyHash> index;
  for (int64_t r = 0; r < m; ++r) index.emplace(g.key[r], r);
  const auto offs = Engine::offsets(d);
  Snew->assign(m * d, 0.0);
  for (int64_t j = 0; j < m; ++j) {
    double num[kMaxD] = {0};
    int64_t den = 0;
    int act = 0;
    for (const auto& v : offs) {
      Key nk = g.key[j];
      for (int c = 0; c < d; ++c) nk[c] += v[c];
      auto it = index.find(nk);
      if (it == index.end()) continue;
      const int64_t r = it->second;
      ++act;
      den += g.cnt[r];
      for (int c = 0; c < d; ++c) num[c] = num[c] + (double)g.cnt[r] * g.S[r * d + c];
    }
    for (int c = 0; c < d; ++c)
      (*Snew)[j * d + c] = act <= 1 ? g.S[j * d + c] : num[c] / (double)den;
  }
}

double ms_dist(const double* a, const double* b, int d) {
  double acc = 0.0;
  for (int c = 0; c < d; ++c) {
    const double t = a[c] - b[c];
    acc = acc + t * t;
  }
  return std::sqrt(acc);
}
}  // namespace

extern "C" {

// mspp_run.  labels n; centroids capacity n*d (first k*d written);
// disp_hist capacity max_iter (per-iteration displacement).
int gso_mspp(const double* X, int64_t n, int32_t d, double h, double tol, int32_t max_iter,
             int32_t* labels, int64_t* k_out, int32_t* iters_out, int32_t* conv_out,
             double* cent_out, double* disp_hist) {
  int st = check_common(n, d, h);
  if (st) return st;
  if (max_iter < 1 || !(tol > 0.0)) return E_INVALID_PARAMETER;
  const int F = fixed_shift(n, h);
  // the first grid: points as particles of count 1
  std::vector<double> pos(X, X + n * d);
  std::vector<int64_t> pc(n, 1), cell_of, root(n);
  for (int64_t p = 0; p < n; ++p)
    for (int c = 0; c < d; ++c)
      if (!std::isfinite(X[p * d + c])) return E_INVALID_INPUT;
  for (int64_t p = 0; p < n; ++p) root[p] = p;  // point -> particle
  MsCells g;
  ms_regrid(pos, pc, d, h, F, &g, &cell_of);
  int it = 0;
  bool conv = false;
  std::vector<double> Snew;
  do {
    ms_jacobi(g, d, &Snew);
    double disp = 0.0;
    const int64_t mp = (int64_t)pc.size();
    for (int64_t i = 0; i < mp; ++i)
      disp = std::max(disp, ms_dist(&Snew[cell_of[i] * d], &pos[i * d], d));
    for (int64_t p = 0; p < n; ++p) root[p] = cell_of[root[p]];  // particle -> its cell
    pos = Snew;  // the cells become the particles (M4)
    pc = g.cnt;
    if (disp_hist) disp_hist[it] = disp;
    ++it;
    if (disp < tol) {
      conv = true;
      break;
    }
    if (it >= max_iter) break;
    ms_regrid(pos, pc, d, h, F, &g, &cell_of);
  } while (true);
  MsCells fin;  // M5: the cells of the final particles
  ms_regrid(pos, pc, d, h, F, &fin, &cell_of);
  for (int64_t p = 0; p < n; ++p) labels[p] = (int32_t)cell_of[root[p]];
  const int64_t k = (int64_t)fin.cnt.size();
  for (int64_t r = 0; r < k * d; ++r) cent_out[r] = fin.S[r];
  *k_out = k;
  *iters_out = it;
  *conv_out = conv ? 1 : 0;
  return OK;
}

}  // extern "C"
