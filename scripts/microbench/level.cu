// One K8 sweep level in isolation: one warp, W lanes each updating one cell from a padded u16
// row list over a Q table (D doubles per row), then __syncwarp.  Cycles per level, variants.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
constexpr int D = 3, MS = 1024;

__device__ __forceinline__ double rs_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double fa = fabs(a);
  if (!(fa < 0x1p+1000) || (fa < 0x1p-900 && a != 0.0)) return __ddiv_rn(a, b);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}

template <int V>
__global__ void __launch_bounds__(512, 1) klevel(const uint16_t* __restrict__ glist, const int* __restrict__ gn,
                                                 int W, int levels, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* Q = (double*)sm;                                   // (2MS+2) rows
  uint16_t* lst = (uint16_t*)(Q + (2 * MS + 2) * D);        // MS * 28
  int* nbn = (int*)(lst + MS * 28);
  double* rden = (double*)(nbn + MS);
  const int tid = threadIdx.x;
  for (int i = tid; i < (2 * MS + 2) * D; i += blockDim.x) Q[i] = 1.0 + (i % 97) * 0.01;
  for (int i = tid; i < MS * 28; i += blockDim.x) lst[i] = glist[i];
  for (int i = tid; i < MS; i += blockDim.x) { nbn[i] = gn[i]; rden[i] = 1.0 / 7.0; }
  __syncthreads();
  if (tid >= 32) return;
  const int lane = tid;
  long long t0 = clock64();
  for (int lev = 0; lev < levels; ++lev) {
    if (lane < W) {
      const int i = (lev * 37 + lane * 13) & (MS - 1);
      const uint2* ls = (const uint2*)(lst + i * 28);
      const int nch = (nbn[i] + 3) >> 2;
      const double dd = 7.0, y = rden[i], ci = 3.0;
      double num[D];
#pragma unroll
      for (int c = 0; c < D; ++c) num[c] = 0.0;
      double va[4][D], vb[4][D];
      auto fetch = [&](double (&v)[4][D], uint2 w) {
        const uint32_t r[4] = {w.x & 0xffffu, w.x >> 16, w.y & 0xffffu, w.y >> 16};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < D; ++c) v[u][c] = Q[r[u] * D + c];
      };
      auto fold = [&](const double (&v)[4][D]) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], v[u][c]);
      };
      if (V == 0 || V == 1) {
        fetch(va, ls[0]);
        for (int ch = 0; ch < nch; ch += 2) {
          fetch(vb, ls[ch + 1]);
          fold(va);
          if (ch + 1 >= nch) break;
          fetch(va, ls[ch + 2]);
          fold(vb);
        }
      } else if (V == 2) {  // all words up front (max 7)
        uint2 wd[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) wd[k] = ls[k];
        fetch(va, wd[0]);
#pragma unroll
        for (int ch = 0; ch < 7; ch += 2) {
          if (ch >= nch) break;
          if (ch + 1 < 7) fetch(vb, wd[ch + 1]);
          fold(va);
          if (ch + 1 >= nch) break;
          if (ch + 2 < 7) fetch(va, wd[ch + 2]);
          fold(vb);
        }
      } else if (V == 3) {  // single buffer
        for (int ch = 0; ch < nch; ++ch) {
          fetch(va, ls[ch]);
          fold(va);
        }
      } else if (V == 4) {  // no loads at all: chain lower bound
        for (int ch = 0; ch < nch; ++ch) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < D; ++c) num[c] = __dadd_rn(num[c], y * (u + 1));
        }
      }
      if (V == 0) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
          const double s1 = rs_div(num[c], dd, y);
          Q[(MS + 1 + i) * D + c] = __dmul_rn(ci, s1);
          Q[i * D + c] = s1;
        }
      } else {  // one guard for all coordinates
        double q0[D], s1[D];
        bool ok = true;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          q0[c] = __dmul_rn(num[c], y);
          const double fa = fabs(num[c]);
          ok &= (fa < 0x1p+1000) && !(fa < 0x1p-900 && num[c] != 0.0);
        }
        if (ok) {
#pragma unroll
          for (int c = 0; c < D; ++c) s1[c] = __fma_rn(__fma_rn(-q0[c], dd, num[c]), y, q0[c]);
        } else {
#pragma unroll
          for (int c = 0; c < D; ++c) s1[c] = __ddiv_rn(num[c], dd);
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
          Q[(MS + 1 + i) * D + c] = __dmul_rn(ci, s1[c]);
          Q[i * D + c] = s1[c];
        }
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { out[0] = t1 - t0; out[1] = (long long)Q[5]; }
}


// lane per (cell, coordinate): 32/D cells per warp
template <int V>
__global__ void __launch_bounds__(512, 1) kcoord(const uint16_t* __restrict__ glist, const int* __restrict__ gn,
                                                 int W, int levels, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* Q = (double*)sm;
  uint16_t* lst = (uint16_t*)(Q + (2 * MS + 2) * D);
  int* nbn = (int*)(lst + MS * 28);
  double* rden = (double*)(nbn + MS);
  const int tid = threadIdx.x;
  for (int i = tid; i < (2 * MS + 2) * D; i += blockDim.x) Q[i] = 1.0 + (i % 97) * 0.01;
  for (int i = tid; i < MS * 28; i += blockDim.x) lst[i] = glist[i];
  for (int i = tid; i < MS; i += blockDim.x) { nbn[i] = gn[i]; rden[i] = 1.0 / 7.0; }
  __syncthreads();
  if (tid >= 32) return;
  constexpr int CPW = 32 / D;
  const int lane = tid, q = lane / D, c = lane - q * D;
  long long t0 = clock64();
  for (int lev = 0; lev < levels; ++lev) {
    if (q < W && q < CPW) {
      const int i = (lev * 37 + q * 13) & (MS - 1);
      const uint2* ls = (const uint2*)(lst + i * 28);
      const int n = nbn[i];
      const int nch = (n + 3) >> 2;
      const double dd = 7.0, y = rden[i], ci = 3.0;
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
      if (V == 0) {  // as in K8 now
        double va[4], vb[4];
        fetch(va, ls[0]);
        for (int ch = 0; ch < nch; ch += 2) {
          fetch(vb, ls[ch + 1]);
          fold(va);
          if (ch + 1 >= nch) break;
          fetch(va, ls[ch + 2]);
          fold(vb);
        }
      } else if (V == 1) {  // words in registers up front, values one chunk ahead, full unroll to 7
        uint2 wd[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) wd[k] = ls[k < 7 ? k : 6];
        double v[7][4];
#pragma unroll
        for (int k = 0; k < 7; ++k) fetch(v[k], wd[k]);
#pragma unroll
        for (int k = 0; k < 7; ++k)
          if (k < nch) fold(v[k]);
      } else if (V == 2) {  // words up front; values fetched one chunk ahead
        uint2 wd[7];
#pragma unroll
        for (int k = 0; k < 7; ++k) wd[k] = ls[k];
        double va[4], vb[4];
        fetch(va, wd[0]);
#pragma unroll
        for (int k = 0; k < 7; k += 2) {
          if (k >= nch) break;
          if (k + 1 < 7) fetch(vb, wd[k + 1]);
          fold(va);
          if (k + 1 >= nch) break;
          if (k + 2 < 7) fetch(va, wd[k + 2]);
          fold(vb);
        }
      } else {  // chain only
        for (int ch = 0; ch < nch; ++ch)
#pragma unroll
          for (int t = 0; t < 4; ++t) num = __dadd_rn(num, y * (t + 1));
      }
      double q0 = __dmul_rn(num, y), s1;
      const double fa = fabs(num);
      if ((fa < 0x1p+1000) && !(fa < 0x1p-900 && num != 0.0))
        s1 = __fma_rn(__fma_rn(-q0, dd, num), y, q0);
      else
        s1 = __ddiv_rn(num, dd);
      Q[(MS + 1 + i) * D + c] = __dmul_rn(ci, s1);
      Q[i * D + c] = s1;
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) { out[0] = t1 - t0; out[1] = (long long)Q[5]; }
}
int main() {
  std::mt19937 rng(1);
  std::vector<uint16_t> L(MS * 28);
  std::vector<int> N(MS);
  for (int i = 0; i < MS; ++i) {
    int n = 10 + rng() % 11;  // 10..20
    N[i] = n;
    int np = (n + 3) & ~3;
    for (int t = 0; t < 28; ++t)
      L[i * 28 + t] = t < n ? (uint16_t)((rng() % 2) ? rng() % MS : MS + 1 + rng() % MS) : (t < np + 4 ? MS : MS);
  }
  uint16_t* gl; int* gn; long long* o;
  cudaMalloc(&gl, L.size() * 2); cudaMalloc(&gn, MS * 4); cudaMalloc(&o, 16);
  cudaMemcpy(gl, L.data(), L.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(gn, N.data(), MS * 4, cudaMemcpyHostToDevice);
  const size_t smem = (2 * MS + 2) * D * 8 + MS * 28 * 2 + MS * 4 + MS * 8;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int W : {1, 5, 10, 19}) {
      long long h[2];
      kern<<<1, 512, smem>>>(gl, gn, W, 200, o);
      kern<<<1, 512, smem>>>(gl, gn, W, 200, o);
      cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("%-28s W=%2d  %7.1f cycles/level  (%s)\n", name, W, h[0] / 200.0,
             cudaGetErrorString(cudaGetLastError()));
    }
  };
  run(kcoord<0>, "C0 coord, K8 now");
  run(kcoord<1>, "C1 coord, all up front");
  run(kcoord<2>, "C2 coord, words up front");
  run(kcoord<3>, "C3 coord, chain only");
  run(klevel<0>, "V0 current");
  run(klevel<1>, "V1 one-guard division");
  run(klevel<2>, "V2 words up front");
  run(klevel<3>, "V3 single buffer");
  run(klevel<4>, "V4 chain only (no loads)");
  return 0;
}
