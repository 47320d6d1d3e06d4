// gridshift.cpp — C++ host API (include/gridshift/gridshift.hpp) over the C-ABI.
//
// Keeps the reference engine signature run(Dataset, EngineConfig) -> ClusterLabeling
// and its exception types (errors.hpp); every call goes to
// the GPU through gs_run.  There is no host compute path.
#include "gridshift/gridshift.hpp"

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

}  // namespace gridshift
