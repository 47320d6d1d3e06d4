// Where do ~400 cycles of per-level overhead come from?  One lane, one level = chain + extras.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double rs_div(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double fa = fabs(a);
  if (!(fa < 0x1p+1000) || (fa < 0x1p-900 && a != 0.0)) return __ddiv_rn(a, b);
  const double r = __fma_rn(-q0, b, a);
  return __fma_rn(r, y, q0);
}
template <int V>
__global__ void k(int levels, int nfix, long long* out, double* res) {
  __shared__ double Q[2048];
  __shared__ int nb[1024];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) Q[i] = 1.0 + i * 1e-3;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) nb[i] = nfix;
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  double acc = 0;
  for (int lev = 0; lev < levels; ++lev) {
    const int i = (lev * 37) & 1023;
    int n = nfix;
    if (V >= 2) n = nb[i];
    double num = 0.0;
    const double y = 1.0 / 7.0;
    if (V == 5) {
#pragma unroll 1
      for (int t = 0; t < n; ++t) num = __dadd_rn(num, 1.0 + t);
    } else {
      const int nch = (n + 3) >> 2;
      for (int ch = 0; ch < nch; ++ch)
#pragma unroll
        for (int t = 0; t < 4; ++t) num = __dadd_rn(num, 1.0 + t);
    }
    double s1 = num;
    if (V >= 1) s1 = rs_div(num, 7.0, y);
    if (V >= 3) { Q[i] = s1; Q[1024 + i] = __dmul_rn(3.0, s1); } else acc += s1;
    if (V >= 4) __syncwarp();
  }
  long long t1 = clock64();
  out[0] = t1 - t0;
  res[0] = acc + Q[3];
}
int main() {
  long long* o; double* r; cudaMalloc(&o, 8); cudaMalloc(&r, 8);
  const char* nm[] = {"chain", "+div", "+nbn load", "+2 STS", "+syncwarp", "plain loop+all"};
  for (int nfix : {4, 12, 20}) {
    auto go = [&](auto kern, int v) {
      long long h;
      kern<<<1, 32>>>(1000, nfix, o, r); kern<<<1, 32>>>(1000, nfix, o, r);
      cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
      printf("n=%2d %-16s %7.1f cycles/level\n", nfix, nm[v], h / 1000.0);
    };
    go(k<0>, 0); go(k<1>, 1); go(k<2>, 2); go(k<3>, 3); go(k<4>, 4); go(k<5>, 5);
  }
  return 0;
}
