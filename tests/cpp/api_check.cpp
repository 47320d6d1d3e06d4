// C++ host API check (include/gridshift/gridshift.hpp): the reference's call shapes
// (gridshift::run, tune_bandwidth, silhouette_subsampled, mspp_run, Tracker) on deterministic
// inputs, printed as JSON for tests/test_cpp_api.py to compare with the CPU oracle, plus the
// errors.hpp exception types of the contract violations.
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "gridshift/gridshift.hpp"

using namespace gridshift;

static Dataset make_points(int n) {  // two groups, deterministic LCG
  Dataset X;
  uint64_t s = 12345;
  auto u = [&]() {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return (double)(s >> 11) * 0x1p-53;
  };
  for (int i = 0; i < n; ++i) {
    const double base = (i % 2) ? 0.7 : 0.2;
    X.push_back({base + 0.08 * u(), base + 0.08 * u()});
  }
  return X;
}

static void print_labeling(const char* name, const Dataset& X, const ClusterLabeling& L) {
  std::printf("{\"what\": \"%s\", \"iterations\": %d, \"k\": %zu, \"labels\": [", name, L.iterations,
              L.centroids.size());
  for (size_t i = 0; i < L.labels.size(); ++i) std::printf(i ? ",%d" : "%d", L.labels[i]);
  std::printf("], \"centroids\": [");
  for (size_t j = 0; j < L.centroids.size(); ++j)
    for (size_t c = 0; c < L.centroids[j].size(); ++c)
      std::printf((j || c) ? ",%.17g" : "%.17g", L.centroids[j][c]);
  std::printf("]}\n");
}

template <typename E, typename F>
static bool throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  const Dataset X = make_points(600);
  std::printf("{\"what\": \"points\", \"X\": [");
  for (size_t i = 0; i < X.size(); ++i) std::printf(i ? ",%.17g,%.17g" : "%.17g,%.17g", X[i][0], X[i][1]);
  std::printf("]}\n");
  print_labeling("run", X, run(X, EngineConfig{0.1, 300, false}));
  print_labeling("mspp", X, mspp_run(X, 0.1, 1e-7, 300));
  const std::vector<double> grid = {0.05, 0.1, 0.2, 0.4};
  const BandwidthSweepResult sw = tune_bandwidth(X, grid, 300, 200, 7);
  std::printf("{\"what\": \"tune\", \"best_h\": %.17g, \"scores\": [", sw.best_h);
  for (size_t i = 0; i < sw.entries.size(); ++i)
    std::printf(i ? ",%.17g" : "%.17g", sw.entries[i].valid ? sw.entries[i].score : -9.0);
  std::printf("]}\n");
  // tracker: a 16 px red square moving +3, +1 px per frame on blue, 8 frames of 96 x 128
  const int T = 8, H = 96, W = 128;
  std::vector<uint8_t> fr((size_t)T * H * W * 3);
  for (int t = 0; t < T; ++t)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        uint8_t* p = &fr[(((size_t)t * H + y) * W + x) * 3];
        const bool in = x >= 30 + 3 * t && x < 46 + 3 * t && y >= 30 + t && y < 46 + t;
        p[0] = in ? 220 : 20;
        p[1] = 20;
        p[2] = in ? 20 : 200;
      }
  Tracker tr(0);
  TrackerConfig tc;
  tc.h = 0.1;
  tr.init(fr.data(), H, W, TrackWindow{37.5, 37.5, 20.0, 20.0}, tc);
  const auto res = tr.track_sequence(fr.data() + (size_t)H * W * 3, T - 1);
  std::printf("{\"what\": \"track\", \"windows\": [");
  for (size_t t = 0; t < res.size(); ++t)
    std::printf(t ? ",%.17g,%.17g,%.17g,%.17g" : "%.17g,%.17g,%.17g,%.17g", res[t].window.ox,
                res[t].window.oy, res[t].window.l, res[t].window.w);
  std::printf("], \"lost\": [");
  for (size_t t = 0; t < res.size(); ++t) std::printf(t ? ",%d" : "%d", res[t].lost ? 1 : 0);
  std::printf("]}\n");
  // contract violations map to the errors.hpp types
  const bool e1 = throws<InvalidBandwidthError>([&] { run(X, EngineConfig{0.0, 10, false}); });
  const bool e2 = throws<EmptyInputError>([&] { run(Dataset{}, EngineConfig{0.1, 10, false}); });
  const bool e3 = throws<InvalidBandwidthError>([&] { tune_bandwidth(X, {0.5, 1.5}); });
  const bool e4 = throws<UndefinedScoreError>(
      [&] { silhouette_subsampled(X, std::vector<int32_t>(X.size(), 0), 100); });
  const bool e5 = throws<TuningFailureError>([&] { tune_bandwidth(Dataset{{0.5, 0.5}}, {0.1}); });
  const bool e6 = throws<InvalidWindowError>(
      [&] { Tracker t2(0); t2.init(fr.data(), H, W, TrackWindow{500, 500, 10, 10}, tc); });
  const bool e7 = throws<InvalidInputError>([&] {
    Dataset bad = X;
    bad[3][1] = 1.0 / 0.0;
    run(bad, EngineConfig{0.1, 10, false});
  });
  std::printf("{\"what\": \"errors\", \"ok\": [%d,%d,%d,%d,%d,%d,%d]}\n", e1, e2, e3, e4, e5, e6, e7);
  return 0;
}
