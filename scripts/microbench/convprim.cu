// Conversion and fp64 primitives of the binning kernel at full occupancy (148 CTAs x 1024
// threads): cycles per warp-instruction per SM.  Each thread runs ITER x U independent chains.
#include <cstdio>
#include <cstdint>

constexpr int ITER = 256, U = 4;

template <int MODE>
__global__ void __launch_bounds__(1024, 1) kc(float* fout, double* dout, long long* cyc, float seed) {
  float f[U];
  double dd[U];
  int ii[U];
  long long ll[U];
  for (int u = 0; u < U; ++u) {
    f[u] = seed + threadIdx.x * 1e-3f + u;
    dd[u] = f[u];
    ii[u] = threadIdx.x + u;
    ll[u] = ii[u];
  }
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) dd[u] = __dadd_rn(dd[u], (double)f[u]);             // F2F.F64.F32 (+DADD)
      if (MODE == 1) dd[u] = __dadd_rn(dd[u], (double)ii[u]);            // I2F.F64 (+DADD)
      if (MODE == 2) dd[u] = __dadd_rn(dd[u], 1.0000001);                // DADD
      if (MODE == 3) dd[u] = __dmul_rn(dd[u], 1.0000001);                // DMUL
      if (MODE == 4) ll[u] += __double2ll_rn(__dadd_rn(dd[u], (double)it)); // F2I.S64.F64 (+DADD)
      if (MODE == 5) ii[u] += __float2int_rz(floorf(__fmul_rn(f[u], 1.01f + it)));  // FMUL FRND F2I
      if (MODE == 6) { f[u] = __fmul_rn(f[u], 1.0001f); }                // FMUL
      if (MODE == 7) ll[u] += __double_as_longlong(__dadd_rn(dd[u] + it, 0x1.8p52));  // magic
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  double s = 0;
  for (int u = 0; u < U; ++u) s += dd[u] + f[u] + ii[u] + (double)ll[u];
  dout[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* fo;
  double* d;
  long long* cyc;
  cudaMalloc(&fo, 148 * 1024 * 4);
  cudaMalloc(&d, 148 * 1024 * 8);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"F2F.F64.F32+DADD", "I2F.F64+DADD", "DADD", "DMUL", "DADD+F2I.S64.F64",
                         "FMUL+FRND+F2I", "FMUL", "DADD(magic)+IADD"};
  auto run = [&](auto kern, int m) {
    long long h[148];
    for (int rep = 0; rep < 2; ++rep) kern<<<148, 1024>>>(fo, d, cyc, 1.5f);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    s /= 148;
    const double winst = 32.0 * ITER * U;  // warp-iterations per SM
    printf("%-22s %8.2f cycles per warp-op per SM  (%6.2f lanes/cycle/SM)\n", names[m], s / winst,
           32.0 * winst / s);
  };
  run(kc<0>, 0); run(kc<1>, 1); run(kc<2>, 2); run(kc<3>, 3); run(kc<4>, 4); run(kc<5>, 5);
  run(kc<6>, 6); run(kc<7>, 7);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
