// DADD dependent-chain latency vs number of concurrently active warps (and active lanes).
#include <cstdio>
__global__ void k(long long* out, int n, int lanes) {
  const int g = threadIdx.x & 31;
  double x = 1.0 + threadIdx.x * 1e-9, y = 1.0000001;
  __syncthreads();
  long long t0 = clock64();
  if (g < lanes)
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  __syncwarp();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  if (x == 12345.0) out[1] = 1;
}
int main() {
  long long* o; long long h[2];
  cudaMalloc(&o, 16);
  for (int lanes : {3, 32})
    for (int T : {32, 128, 256, 512, 1024}) {
      k<<<1, T>>>(o, 2048, lanes); k<<<1, T>>>(o, 2048, lanes);
      cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
      printf("lanes=%2d warps=%2d: %6.2f cycles per dependent DADD\n", lanes, T / 32, h[0] / 2048.0);
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
