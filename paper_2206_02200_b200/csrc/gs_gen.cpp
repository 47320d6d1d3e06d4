// gs_gen.cpp — seeded synthetic inputs for the five BASELINE.json configs.
//
// Host-side generation with a counter-based SplitMix64 stream and fp64 Box-Muller normals, so
// the GPU engine and the CPU oracle consume identical bytes.  The paper's evaluation sets
// (UCI sensor sets, BSDS500, OTB100) are not in this container; these seeded generators stand
// in for them with the shapes, sizes and value distributions BASELINE.json names.  Every value
// depends only on (seed, stream, counter), so parallel generation is deterministic.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Counter-based stream: value #i of stream s under seed.
struct Stream {
  uint64_t key;
  Stream(uint64_t seed, uint64_t s) : key(mix64(seed ^ mix64(s + 0x5851F42D4C957F2Dull))) {}
  uint64_t u64(uint64_t i) const { return mix64(key + i * 0x9E3779B97F4A7C15ull); }
  double u01(uint64_t i) const { return (double)(u64(i) >> 11) * 0x1.0p-53; }  // [0,1)
  double uab(uint64_t i, double a, double b) const { return a + (b - a) * u01(i); }
  // Box-Muller normal pair from counters (2i, 2i+1); u1 in (0,1].
  void normal2(uint64_t i, double* z0, double* z1) const {
    double u1 = 1.0 - u01(2 * i);
    double u2 = u01(2 * i + 1);
    double r = std::sqrt(-2.0 * std::log(u1));
    double t = 6.283185307179586476925286766559 * u2;
    *z0 = r * std::cos(t);
    *z1 = r * std::sin(t);
  }
  double normal(uint64_t i) const {
    double a, b;
    normal2(i, &a, &b);
    return a;
  }
};


// Deterministic parallel loop: every iteration depends only on its index.
template <typename F>
void par_for(int64_t n, F fn) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 64) nt = 64;
  if (n < 65536) nt = 1;
  std::vector<std::thread> th;
  int64_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    int64_t a = (int64_t)t * chunk, b = std::min<int64_t>(n, a + chunk);
    if (a >= b) break;
    th.emplace_back([=, &fn] { for (int64_t i = a; i < b; ++i) fn(i); });
  }
  for (auto& x : th) x.join();
}

inline double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

}  // namespace

extern "C" {

// cfg1: k isotropic Gaussian blobs in d dims, centres U[lo,hi]^d, exactly n/k points each
// (remainder to the first blobs), then a seeded Fisher-Yates shuffle.  fp64 output n x d.
int gsgen_blobs(uint64_t seed, int64_t n, int32_t d, int32_t k, double sigma, double lo,
                double hi, double* out) {
  if (n < 0 || d < 1 || k < 1) return 1;
  Stream sc(seed, 1), sp(seed, 2), sh(seed, 3);
  std::vector<double> centres((size_t)k * d);
  for (int64_t i = 0; i < (int64_t)k * d; ++i) centres[i] = sc.uab(i, lo, hi);
  par_for(n, [&](int64_t p) {
    int64_t per = n / k, rem = n % k;
    // blob b owns points [start_b, start_b + per + (b < rem))
    int64_t b = (p < rem * (per + 1)) ? p / (per + 1) : rem + (p - rem * (per + 1)) / per;
    for (int c = 0; c < d; ++c)
      out[p * d + c] = centres[b * d + c] + sigma * sp.normal((uint64_t)p * d + c);
  });
  for (int64_t i = n - 1; i > 0; --i) {  // Fisher-Yates
    int64_t j = (int64_t)(sh.u64(i) % (uint64_t)(i + 1));
    for (int c = 0; c < d; ++c) std::swap(out[i * d + c], out[j * d + c]);
  }
  return 0;
}

// cfg2: W x H image of `sites` Voronoi regions (sites uniform over the pixel domain, Euclidean,
// ties -> lower index), each a uniform random colour, plus N(0, sigma^2) per channel, clipped to
// [0,1].  Features (r,g,b), row-major pixel order kept.  fp32 output (W*H) x 3.
int gsgen_voronoi_rgb(uint64_t seed, int32_t W, int32_t H, int32_t sites, double sigma,
                      float* out) {
  if (W < 1 || H < 1 || sites < 1) return 1;
  Stream ss(seed, 1), sc(seed, 2), sn(seed, 3);
  std::vector<double> sx(sites), sy(sites), col((size_t)sites * 3);
  for (int s = 0; s < sites; ++s) {
    sx[s] = ss.uab(2 * s, 0.0, (double)W);
    sy[s] = ss.uab(2 * s + 1, 0.0, (double)H);
    for (int c = 0; c < 3; ++c) col[s * 3 + c] = sc.u01(s * 3 + c);
  }
  par_for((int64_t)W * H, [&](int64_t p) {
    double px = (double)(p % W) + 0.5, py = (double)(p / W) + 0.5;
    int best = 0;
    double bd = 1e300;
    for (int s = 0; s < sites; ++s) {
      double dx = px - sx[s], dy = py - sy[s], dd = dx * dx + dy * dy;
      if (dd < bd) { bd = dd; best = s; }
    }
    double z[4];
    sn.normal2((uint64_t)p * 2, &z[0], &z[1]);
    sn.normal2((uint64_t)p * 2 + 1, &z[2], &z[3]);
    for (int c = 0; c < 3; ++c) out[p * 3 + c] = (float)clip01(col[best * 3 + c] + sigma * z[c]);
  });
  return 0;
}

// cfg3: W x H image of `sites` Voronoi regions with linear colour gradients:
// colour = base U[0,1]^3 + G (p - site) / (W, H), G in U[-grad, grad]^{3x2}, + N(0, sigma^2),
// clipped.  Features (x/W, y/H, r, g, b) as BASELINE.json states.  fp32 output (W*H) x 5.
int gsgen_voronoi_rgbxy(uint64_t seed, int32_t W, int32_t H, int32_t sites, double grad,
                        double sigma, float* out) {
  if (W < 1 || H < 1 || sites < 1) return 1;
  Stream ss(seed, 1), sc(seed, 2), sg(seed, 4), sn(seed, 3);
  std::vector<double> sx(sites), sy(sites), col((size_t)sites * 3), G((size_t)sites * 6);
  for (int s = 0; s < sites; ++s) {
    sx[s] = ss.uab(2 * s, 0.0, (double)W);
    sy[s] = ss.uab(2 * s + 1, 0.0, (double)H);
    for (int c = 0; c < 3; ++c) col[s * 3 + c] = sc.u01(s * 3 + c);
    for (int c = 0; c < 6; ++c) G[s * 6 + c] = sg.uab(s * 6 + c, -grad, grad);
  }
  par_for((int64_t)W * H, [&](int64_t p) {
    int64_t xi = p % W, yi = p / W;
    double px = (double)xi + 0.5, py = (double)yi + 0.5;
    int best = 0;
    double bd = 1e300;
    for (int s = 0; s < sites; ++s) {
      double dx = px - sx[s], dy = py - sy[s], dd = dx * dx + dy * dy;
      if (dd < bd) { bd = dd; best = s; }
    }
    double rx = (px - sx[best]) / W, ry = (py - sy[best]) / H;
    double z[4];
    sn.normal2((uint64_t)p * 2, &z[0], &z[1]);
    sn.normal2((uint64_t)p * 2 + 1, &z[2], &z[3]);
    out[p * 5 + 0] = (float)((double)xi / W);
    out[p * 5 + 1] = (float)((double)yi / H);
    for (int c = 0; c < 3; ++c) {
      double v = col[best * 3 + c] + G[best * 6 + c * 2] * rx + G[best * 6 + c * 2 + 1] * ry;
      out[p * 5 + 2 + c] = (float)clip01(v + sigma * z[c]);
    }
  });
  return 0;
}

// cfg4: a video of W x H frames with `ne` axis-aligned solid-colour ellipses (colour U[0,1]^3,
// semi-axes U[amin,amax] px, initial centre uniform over the frame, velocity U[-vmax,vmax]^2
// px/frame reflecting at the borders, z-order by index) on a background of base colour
// U[0,1]^3 + N(0, bg_sigma^2) per pixel, clipped.  Writes frames [f0, f0+nf) as fp32
// (nf*W*H) x 3; any frame subset is identical to the same frames of the full sequence.
int gsgen_ellipse_frames(uint64_t seed, int32_t W, int32_t H, int32_t ne, double amin,
                         double amax, double vmax, double bg_sigma, int64_t f0, int64_t nf,
                         float* out) {
  if (W < 1 || H < 1 || ne < 0 || f0 < 0 || nf < 0) return 1;
  Stream se(seed, 1), sb(seed, 2), sn(seed, 3);
  std::vector<double> col((size_t)ne * 3), ax(ne), ay(ne), cx0(ne), cy0(ne), vx(ne), vy(ne);
  for (int e = 0; e < ne; ++e) {
    uint64_t b = (uint64_t)e * 16;
    for (int c = 0; c < 3; ++c) col[e * 3 + c] = se.u01(b + c);
    ax[e] = se.uab(b + 3, amin, amax);
    ay[e] = se.uab(b + 4, amin, amax);
    cx0[e] = se.uab(b + 5, 0.0, (double)W);
    cy0[e] = se.uab(b + 6, 0.0, (double)H);
    vx[e] = se.uab(b + 7, -vmax, vmax);
    vy[e] = se.uab(b + 8, -vmax, vmax);
  }
  double bg[3];
  for (int c = 0; c < 3; ++c) bg[c] = sb.u01(c);
  auto reflect = [](double p0, double v, double t, double L) {
    // position of a point moving at v from p0, reflecting in [0, L]
    double p = p0 + v * t;
    double period = 2.0 * L;
    double r = std::fmod(p, period);
    if (r < 0) r += period;
    return r <= L ? r : period - r;
  };
  for (int64_t f = f0; f < f0 + nf; ++f) {
    std::vector<double> cx(ne), cy(ne);
    for (int e = 0; e < ne; ++e) {
      cx[e] = reflect(cx0[e], vx[e], (double)f, (double)W);
      cy[e] = reflect(cy0[e], vy[e], (double)f, (double)H);
    }
    float* fo = out + (f - f0) * (int64_t)W * H * 3;
    const uint64_t fbase = (uint64_t)f * (uint64_t)W * H;
    par_for((int64_t)W * H, [&](int64_t p) {
      double px = (double)(p % W) + 0.5, py = (double)(p / W) + 0.5;
      int top = -1;
      for (int e = 0; e < ne; ++e) {
        double dx = (px - cx[e]) / ax[e], dy = (py - cy[e]) / ay[e];
        if (dx * dx + dy * dy <= 1.0) top = e;  // later index is drawn on top
      }
      if (top >= 0) {
        for (int c = 0; c < 3; ++c) fo[p * 3 + c] = (float)col[top * 3 + c];
      } else {
        double z[4];
        sn.normal2((fbase + p) * 2, &z[0], &z[1]);
        sn.normal2((fbase + p) * 2 + 1, &z[2], &z[3]);
        for (int c = 0; c < 3; ++c) fo[p * 3 + c] = (float)clip01(bg[c] + bg_sigma * z[c]);
      }
    });
  }
  return 0;
}

// cfg5: n points from a mixture of `k` axis-aligned 3-D Gaussians: centres U[lo,hi]^3, per-axis
// sigma U[smin,smax], weights Dirichlet(1) (normalised Exp(1) draws); each point draws its
// component independently (so counts are multinomial(n, w) and the order is already random).
// Points [p0, p0+np) of the full sequence are written as fp32 np x 3.
int gsgen_gmm3(uint64_t seed, int64_t p0, int64_t np, int32_t k, double lo, double hi,
               double smin, double smax, float* out) {
  if (k < 1 || p0 < 0 || np < 0) return 1;
  Stream sc(seed, 1), sw(seed, 2), sz(seed, 3), sp(seed, 4);
  std::vector<double> mu((size_t)k * 3), sg((size_t)k * 3), cdf(k);
  double tot = 0.0;
  for (int j = 0; j < k; ++j) {
    for (int c = 0; c < 3; ++c) {
      mu[j * 3 + c] = sc.uab(j * 3 + c, lo, hi);
      sg[j * 3 + c] = sc.uab(1000 + j * 3 + c, smin, smax);
    }
    double e = -std::log(1.0 - sw.u01(j));
    tot += e;
    cdf[j] = tot;
  }
  for (int j = 0; j < k; ++j) cdf[j] /= tot;
  par_for(np, [&](int64_t q) {
    uint64_t p = (uint64_t)(p0 + q);
    double u = sz.u01(p);
    int j = 0;
    while (j < k - 1 && u >= cdf[j]) ++j;
    double z[4];
    sp.normal2(p * 2, &z[0], &z[1]);
    sp.normal2(p * 2 + 1, &z[2], &z[3]);
    for (int c = 0; c < 3; ++c) out[q * 3 + c] = (float)(mu[j * 3 + c] + sg[j * 3 + c] * z[c]);
  });
  return 0;
}

}  // extern "C"
