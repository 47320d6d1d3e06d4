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

}  // namespace gridshift
