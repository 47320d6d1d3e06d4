// Binning primitives at full occupancy (148 CTAs x 768 threads, one per SM): cycles per
// warp-instruction per SM for the operations K2 is built from.  Each test runs ITER
// iterations of U independent ops per thread; cycles = SM-average clock64 span.
#include <cstdio>
#include <cstdint>

constexpr int ITER = 256, U = 4;

__device__ __forceinline__ unsigned hashl(unsigned i, unsigned salt) { return (i * 2654435761u + salt * 40503u) >> 20; }

template <int MODE>
__global__ void __launch_bounds__(768, 1) kb(unsigned* gout, unsigned long long* gtab, long long* cyc, unsigned salt) {
  __shared__ unsigned tab[4096 * 2];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  unsigned acc = threadIdx.x;
  double dacc = threadIdx.x * 1e-3;
  const unsigned lane = threadIdx.x & 31;
  long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned a = (hashl(threadIdx.x + 768 * (it * U + u), salt) & 4095);
      if (MODE == 0) atomicAdd(&tab[a], 1u);                     // ATOMS spread, no return
      if (MODE == 1) acc += atomicAdd(&tab[a], acc);             // ATOMS spread, return used
      if (MODE == 2) atomicAdd(&tab[(a & 7) * 512 + 0], 1u);     // ATOMS 8 hot addresses
      if (MODE == 3) { unsigned v = tab[a]; tab[a] = v + acc; }  // plain LDS+STS (races ok)
      if (MODE == 4) acc += __match_any_sync(0xffffffffu, a & 15);
      if (MODE == 5) acc += __reduce_add_sync(0xffffffffu, a);
      if (MODE == 6) dacc = __dmul_rn(dacc, 1.0000001);
      if (MODE == 7) atomicAdd(&gtab[(blockIdx.x * 4096 + a)], 1ull);  // REDG.64 spread
      if (MODE == 8) acc += __ballot_sync(0xffffffffu, a & 1);
      if (MODE == 9) atomicAdd(&tab[threadIdx.x * 5 & 4095], 1u);       // conflict-free banks
      if (MODE == 10) acc += __match_any_sync(0xffffffffu, (lane >> 3) + it);  // 4 groups
      if (MODE == 11) acc += __shfl_sync(0xffffffffu, acc, a & 31);
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  gout[blockIdx.x * blockDim.x + threadIdx.x] = acc + tab[threadIdx.x] + (unsigned)dacc;
}

int main() {
  unsigned* go;
  unsigned long long* gt;
  long long* cyc;
  cudaMalloc(&go, 148 * 768 * 4);
  cudaMalloc(&gt, 148 * 4096 * 8);
  cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"ATOMS spread no-ret", "ATOMS spread ret-used", "ATOMS 8 hot addr",
                         "LDS+STS spread", "MATCH.ANY (16 grp)", "REDUX.SUM", "DMUL",
                         "REDG.64 spread", "VOTE.BALLOT", "ATOMS bank-free", "MATCH.ANY (4 grp)",
                         "SHFL.IDX"};
  auto run = [&](auto kern, int m) {
    long long h[148];
    for (int rep = 0; rep < 2; ++rep) kern<<<148, 768>>>(go, gt, cyc, 7);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    s /= 148;
    const double winst = 24.0 * ITER * U;  // warp-instructions per SM
    printf("%-22s %8.2f cycles per warp-op per SM  (%6.2f lanes/cycle/SM)\n", names[m], s / winst,
           32.0 * winst / s);
  };
  run(kb<0>, 0); run(kb<1>, 1); run(kb<2>, 2); run(kb<3>, 3); run(kb<4>, 4); run(kb<5>, 5);
  run(kb<6>, 6); run(kb<7>, 7); run(kb<8>, 8); run(kb<9>, 9); run(kb<10>, 10); run(kb<11>, 11);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
