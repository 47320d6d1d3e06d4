// gridshift.hpp — C++ host API of the B200-native GridShift engine.
//
// Mirrors the reference's engine module:
//   ClusterLabeling run(const Dataset& X, const EngineConfig& cfg)
// with EngineConfig and ClusterLabeling.  Errors are the
// errors.hpp exceptions; non-convergence is a flagged partial result, not an exception
// (SPEC.md:139).  The work runs on the GPU through the C-ABI in gridshift_c.h.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "gridshift/errors.hpp"
#include "gridshift_c.h"

namespace gridshift {

using FeatureVector = std::vector<double>;
using Dataset = std::vector<FeatureVector>;  // n FeatureVectors of uniform dimension d

struct EngineConfig {
  double h = 0.0;
  int max_iterations = 1000;
  bool record_history = false;
};

struct HistoryEntry {
  int64_t m;                 // active cells entering the iteration
  double max_displacement;   // max Euclidean centroid displacement of the sweep
};

struct ClusterLabeling {
  std::vector<int32_t> labels;          // per point, 0..k-1 (lexicographic rank of final cell)
  std::vector<FeatureVector> centroids; // per cluster
  int iterations = 0;
  bool converged = true;                // false: max_iterations reached (warning flag)
  std::vector<HistoryEntry> history;    // filled when record_history
};

// Throws the errors.hpp type that `status` maps to (no-op for GS_OK).
void throw_for_status(gs_status status, const char* detail);

// A reusable engine bound to one device (owns device buffers and a stream).
class Engine {
 public:
  explicit Engine(int device = 0);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  ClusterLabeling run(const Dataset& X, const EngineConfig& cfg);
  // Flat row-major n x d input (float or double), optionally already on the device.
  ClusterLabeling run(const float* X, int64_t n, int32_t d, const EngineConfig& cfg,
                      bool on_device = false);
  ClusterLabeling run(const double* X, int64_t n, int32_t d, const EngineConfig& cfg,
                      bool on_device = false);
  // Independent frames [batch][n][d], one labeling per frame.
  std::vector<ClusterLabeling> run_batch(const float* X, int64_t batch, int64_t n, int32_t d,
                                         const EngineConfig& cfg, bool on_device = false);

  gs_ctx* handle() { return ctx_; }

 private:
  std::vector<ClusterLabeling> run_raw(const void* X, int32_t dtype, int64_t batch, int64_t n,
                                       int32_t d, const EngineConfig& cfg, bool on_device);
  gs_ctx* ctx_ = nullptr;
};

// engine.run on device 0 with a process-wide engine.
ClusterLabeling run(const Dataset& X, const EngineConfig& cfg);

// ---- metrics module: the bandwidth sweep, scored by silhouette_subsampled
struct SweepEntry {  // one (h, silhouette score, cluster count) pair
  double h = 0.0;
  double score = 0.0;   // meaningful when valid
  bool valid = false;   // false: < 2 clusters in the sample (undefined, skipped)
  int64_t clusters = 0;
  int iterations = 0;
};
struct BandwidthSweepResult {
  std::vector<SweepEntry> entries;
  double best_h = 0.0;
};
// tune_bandwidth(X, clusterer = the GPU engine, h_grid); throws
// TuningFailureError when no entry is scorable, InvalidBandwidthError for h outside (0, 1].
BandwidthSweepResult tune_bandwidth(const Dataset& X, const std::vector<double>& h_grid,
                                    int max_iterations = 1000, int64_t cap = 10000,
                                    uint64_t seed = 0, int max_concurrent = 8);
// silhouette_subsampled(X, labels, cap, seed); UndefinedScoreError for < 2
// clusters in the sample.
double silhouette_subsampled(const Dataset& X, const std::vector<int32_t>& labels, int64_t cap,
                             uint64_t seed = 0);

// ---- baselines module: MS++ (SPEC.md:197-203), parallel grid mean shift on the GPU
ClusterLabeling mspp_run(const Dataset& X, double h, double tol, int max_iterations = 300);

// ---- tracker module (Algorithm 2)
struct TrackWindow {  // W(o, l, w)
  double ox = 0.0, oy = 0.0, l = 0.0, w = 0.0;
};
struct TrackerConfig {  // SPEC.md:448-451 with the ledger defaults (:490-494)
  double h = 0.0;
  double f = 1.0;
  double eta = 1.0;
  int max_inner_iters = 20;
  int engine_max_iterations = 1000;
  int top_k = 1;
  std::vector<int32_t> ids;  // explicit cluster ids (overrides top_k)
};
struct TrackResult {  // per tracked frame: the emitted window and the lost-target flag
  TrackWindow window;
  bool lost = false;
  int inner_iterations = 0;
};
class Tracker {
 public:
  explicit Tracker(int device = 0);
  ~Tracker();
  Tracker(const Tracker&) = delete;
  Tracker& operator=(const Tracker&) = delete;
  // init_tracker on an H x W x 3 8-bit RGB frame; returns the cluster count
  int64_t init(const uint8_t* frame0, int H, int W, const TrackWindow& window,
               const TrackerConfig& cfg);
  // track_sequence over T frames (T x H x W x 3), continuing the state
  std::vector<TrackResult> track_sequence(const uint8_t* frames, int64_t T);

 private:
  gs_tracker* t_ = nullptr;
};


}  // namespace gridshift
