// Isolate: DADD latency with register operands, 1 lane vs 32 lanes; divergence+syncwarp cost.
#include <cstdio>
__global__ void k(long long* out, int variant, int n) {
  __shared__ double s[1024];
  const int g = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + i * 1e-6;
  __syncthreads();
  double x = s[g], y = s[g + 32];
  long long t0 = clock64(), t1;
  if (variant == 0) {           // all lanes: register chain
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
  } else if (variant == 1) {    // 3 lanes (divergent) register chain
    if (g < 3) for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
    __syncwarp();
  } else if (variant == 2) {    // all lanes: smem operand per add (independent loads)
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, s[(i * 8 + g) & 1023]);
  } else if (variant == 3) {    // 3 lanes: smem operand per add
    if (g < 3) for (int i = 0; i < n; ++i) x = __dadd_rn(x, s[(i * 8 + g) & 1023]);
    __syncwarp();
  } else if (variant == 4) {    // empty divergent region + syncwarp, n times
    for (int i = 0; i < n; ++i) { if (g < 3) x = __dadd_rn(x, y); __syncwarp(); }
  } else {                      // unrolled-by-8 preload then adds, all lanes
    for (int i = 0; i < n; i += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = s[((i + u) * 8 + g) & 1023];
#pragma unroll
      for (int u = 0; u < 8; ++u) x = __dadd_rn(x, v[u]);
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = (long long)x; }
}
int main() {
  long long* o; long long h[2];
  cudaMalloc(&o, 16);
  const char* names[] = {"reg chain 32 lanes", "reg chain 3 lanes", "smem operand 32 lanes",
                         "smem operand 3 lanes", "divergent add+syncwarp per step", "preload8 32 lanes"};
  for (int v = 0; v < 6; ++v) {
    k<<<1, 32>>>(o, v, 512); k<<<1, 32>>>(o, v, 512);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("%-34s %6.2f cycles/step\n", names[v], h[0] / 512.0);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
