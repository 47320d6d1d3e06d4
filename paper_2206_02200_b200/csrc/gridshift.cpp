// gridshift.cpp — C++ host API (include/gridshift/gridshift.hpp) over the C-ABI.
//
// Keeps the reference engine signature run(Dataset, EngineConfig) -> ClusterLabeling
// and its exception types (errors.hpp); every call goes to
// the GPU through gs_run.  There is no host compute path.
#include "gridshift/gridshift.hpp"

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>

namespace gridshift {

void throw_for_status(gs_status s, const char* detail) {
  if (s == GS_OK) return;
  std::string msg = std::string(gs_status_string(s)) + (detail && *detail ? ": " : "") +
                    (detail ? detail : "");
  switch (s) {
    case GS_E_INVALID_INPUT: throw InvalidInputError(msg);
    case GS_E_INVALID_BANDWIDTH: throw InvalidBandwidthError(msg);
    case GS_E_EMPTY_INPUT: throw EmptyInputError(msg);
    case GS_E_INVALID_PARAMETER: throw InvalidParameterError(msg);
    case GS_E_KEY_RANGE: throw InvalidParameterError(msg);
    case GS_E_INTERNAL_INVARIANT: throw InternalInvariantError(msg);
    case GS_E_TUNING_FAILED: throw TuningFailureError(msg);
    case GS_E_UNDEFINED_SCORE: throw UndefinedScoreError(msg);
    case GS_E_INVALID_WINDOW: throw InvalidWindowError(msg);
    case GS_E_SELECTION: throw SelectionError(msg);
    default: throw Error(msg);
  }
}

Engine::Engine(int device) {
  gs_status s = gs_create(device, nullptr, &ctx_);
  throw_for_status(s, "gs_create");
}

Engine::~Engine() { gs_destroy(ctx_); }

std::vector<ClusterLabeling> Engine::run_raw(const void* X, int32_t dtype, int64_t batch,
                                             int64_t n, int32_t d, const EngineConfig& cfg,
                                             bool on_device) {
  gs_input in{X, n, d, dtype, batch, on_device ? 1 : 0, 0};
  gs_config c{cfg.h, cfg.max_iterations, cfg.record_history ? GS_RECORD_HISTORY : 0u};
  gs_status v = gs_validate(&in, &c);
  throw_for_status(v, "");
  std::vector<int32_t> labels((size_t)(batch * n));
  std::vector<int64_t> k(batch);
  std::vector<int32_t> iters(batch), conv(batch);
  gs_result r{labels.data(), k.data(), iters.data(), conv.data()};
  gs_status s = gs_run(ctx_, &in, &c, &r);
  throw_for_status(s, gs_last_error(ctx_));
  std::vector<ClusterLabeling> out(batch);
  for (int64_t f = 0; f < batch; ++f) {
    ClusterLabeling& L = out[f];
    L.labels.assign(labels.begin() + f * n, labels.begin() + (f + 1) * n);
    L.iterations = iters[f];
    L.converged = conv[f] != 0;
    std::vector<double> cent((size_t)(k[f] * d));
    throw_for_status(gs_get_centroids(ctx_, f, cent.data(), k[f]), gs_last_error(ctx_));
    L.centroids.resize(k[f]);
    for (int64_t j = 0; j < k[f]; ++j)
      L.centroids[j].assign(cent.begin() + j * d, cent.begin() + (j + 1) * d);
    if (cfg.record_history) {
      std::vector<int64_t> m(iters[f]);
      std::vector<double> disp(iters[f]);
      throw_for_status(gs_get_history(ctx_, f, m.data(), disp.data(), iters[f]),
                       gs_last_error(ctx_));
      for (int t = 0; t < iters[f]; ++t) L.history.push_back({m[t], disp[t]});
    }
  }
  return out;
}

ClusterLabeling Engine::run(const Dataset& X, const EngineConfig& cfg) {
  if (X.empty()) throw EmptyInputError("empty dataset");
  const size_t d = X[0].size();
  if (d == 0) throw InvalidParameterError("zero-dimensional feature vectors");
  std::vector<double> flat;
  flat.reserve(X.size() * d);
  for (const auto& x : X) {
    if (x.size() != d) throw InvalidInputError("feature vectors of differing dimension");
    flat.insert(flat.end(), x.begin(), x.end());
  }
  return run(flat.data(), (int64_t)X.size(), (int32_t)d, cfg, false);
}

ClusterLabeling Engine::run(const float* X, int64_t n, int32_t d, const EngineConfig& cfg,
                            bool on_device) {
  return std::move(run_raw(X, GS_F32, 1, n, d, cfg, on_device)[0]);
}

ClusterLabeling Engine::run(const double* X, int64_t n, int32_t d, const EngineConfig& cfg,
                            bool on_device) {
  return std::move(run_raw(X, GS_F64, 1, n, d, cfg, on_device)[0]);
}

std::vector<ClusterLabeling> Engine::run_batch(const float* X, int64_t batch, int64_t n,
                                               int32_t d, const EngineConfig& cfg,
                                               bool on_device) {
  return run_raw(X, GS_F32, batch, n, d, cfg, on_device);
}

ClusterLabeling run(const Dataset& X, const EngineConfig& cfg) {
  // validate before touching the device so contract errors need no GPU
  if (!(cfg.h > 0.0) || !std::isfinite(cfg.h)) throw InvalidBandwidthError("h must be > 0");
  if (X.empty()) throw EmptyInputError("empty dataset");
  static std::mutex mu;
  static Engine* engine = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!engine) engine = new Engine(0);
  return engine->run(X, cfg);
}

namespace {
std::vector<double> flatten(const Dataset& X, int32_t* d_out) {
  if (X.empty()) throw EmptyInputError("empty dataset");
  const size_t d = X[0].size();
  if (d == 0) throw InvalidParameterError("zero-dimensional feature vectors");
  std::vector<double> flat;
  flat.reserve(X.size() * d);
  for (const auto& x : X) {
    if (x.size() != d) throw InvalidInputError("feature vectors of differing dimension");
    flat.insert(flat.end(), x.begin(), x.end());
  }
  *d_out = (int32_t)d;
  return flat;
}

struct TunerHandle {
  gs_tuner* t = nullptr;
  explicit TunerHandle(int conc) { throw_for_status(gs_tuner_create(0, conc, &t), "gs_tuner_create"); }
  ~TunerHandle() { gs_tuner_destroy(t); }
};
}  // namespace

BandwidthSweepResult tune_bandwidth(const Dataset& X, const std::vector<double>& h_grid,
                                    int max_iterations, int64_t cap, uint64_t seed,
                                    int max_concurrent) {
  int32_t d;
  std::vector<double> flat = flatten(X, &d);
  TunerHandle th(std::max(1, max_concurrent));
  gs_input in{flat.data(), (int64_t)X.size(), d, GS_F64, 1, 0, 0};
  std::vector<gs_sweep_entry> e(std::max<size_t>(1, h_grid.size()));
  double best = 0.0;
  throw_for_status(gs_tune_bandwidth(th.t, &in, h_grid.data(), (int32_t)h_grid.size(),
                                     max_iterations, cap, seed, e.data(), &best),
                   gs_tuner_last_error(th.t));
  BandwidthSweepResult r;
  r.best_h = best;
  for (size_t i = 0; i < h_grid.size(); ++i)
    r.entries.push_back({e[i].h, e[i].score, e[i].valid != 0, e[i].k, e[i].iterations});
  return r;
}

double silhouette_subsampled(const Dataset& X, const std::vector<int32_t>& labels, int64_t cap,
                             uint64_t seed) {
  int32_t d;
  std::vector<double> flat = flatten(X, &d);
  if (labels.size() != X.size()) throw InvalidInputError("one label per point");
  TunerHandle th(1);
  gs_input in{flat.data(), (int64_t)X.size(), d, GS_F64, 1, 0, 0};
  double score = 0.0;
  throw_for_status(gs_silhouette_subsampled(th.t, &in, labels.data(), 0, cap, seed, &score),
                   gs_tuner_last_error(th.t));
  return score;
}

ClusterLabeling mspp_run(const Dataset& X, double h, double tol, int max_iterations) {
  int32_t d;
  std::vector<double> flat = flatten(X, &d);
  Engine eng(0);
  gs_input in{flat.data(), (int64_t)X.size(), d, GS_F64, 1, 0, 0};
  std::vector<int32_t> labels(X.size());
  int64_t k = 0;
  int32_t it = 0, cv = 0;
  gs_result r{labels.data(), &k, &it, &cv};
  std::vector<double> disp((size_t)std::max(1, max_iterations));
  throw_for_status(gs_mspp_run(eng.handle(), &in, h, tol, max_iterations, &r, disp.data()),
                   gs_last_error(eng.handle()));
  ClusterLabeling L;
  L.labels = std::move(labels);
  L.iterations = it;
  L.converged = cv != 0;
  std::vector<double> cent((size_t)(k * d));
  throw_for_status(gs_get_centroids(eng.handle(), 0, cent.data(), k), gs_last_error(eng.handle()));
  L.centroids.resize(k);
  for (int64_t j = 0; j < k; ++j) L.centroids[j].assign(cent.begin() + j * d, cent.begin() + (j + 1) * d);
  for (int t = 0; t < it; ++t) L.history.push_back({0, disp[t]});  // MS++ displacement per iteration
  return L;
}

Tracker::Tracker(int device) { throw_for_status(gs_tracker_create(device, &t_), "gs_tracker_create"); }

Tracker::~Tracker() { gs_tracker_destroy(t_); }

int64_t Tracker::init(const uint8_t* frame0, int H, int W, const TrackWindow& w,
                      const TrackerConfig& cfg) {
  gs_window gw{w.ox, w.oy, w.l, w.w};
  gs_tracker_config c{cfg.h, cfg.f, cfg.eta, cfg.max_inner_iters, cfg.engine_max_iterations,
                      cfg.top_k, (int32_t)cfg.ids.size(), cfg.ids.empty() ? nullptr : cfg.ids.data()};
  int64_t k = 0;
  throw_for_status(gs_track_init(t_, frame0, H, W, 0, &gw, &c, &k), gs_tracker_last_error(t_));
  return k;
}

std::vector<TrackResult> Tracker::track_sequence(const uint8_t* frames, int64_t T) {
  std::vector<gs_window> out((size_t)std::max<int64_t>(T, 1));
  std::vector<int32_t> lost((size_t)std::max<int64_t>(T, 1)), inner((size_t)std::max<int64_t>(T, 1));
  throw_for_status(gs_track_sequence(t_, frames, T, 0, out.data(), lost.data(), inner.data()),
                   gs_tracker_last_error(t_));
  std::vector<TrackResult> r((size_t)T);
  for (int64_t t = 0; t < T; ++t)
    r[t] = TrackResult{{out[t].ox, out[t].oy, out[t].l, out[t].w}, lost[t] != 0, inner[t]};
  return r;
}

}  // namespace gridshift
