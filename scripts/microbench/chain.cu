// Why does K8's ordered add chain cost ~75 cycles/add?  Variants of the same pattern.
#include <cstdio>
#include <cstdint>
constexpr int G = 32, D = 3;
__global__ void kchain(long long* out, int len, int variant, int park) {
  __shared__ double stg[D * G * 16];
  const int tid = threadIdx.x, g = tid & 31, w = tid >> 5;
  for (int i = tid; i < D * G * 16; i += blockDim.x) stg[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  if (park && w > 0) {  // other warps wait on a named barrier, like K8's idle warps
    asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
    return;
  }
  if (w != 0) return;
  double num = 0.0;
  long long t0 = clock64();
  for (int rep = 0; rep < 16; ++rep) {
    if (g < D) {
      if (variant == 0) {  // K8 today: chunks of 8 preloads, predicated adds
        for (int u0 = 0; u0 < len; u0 += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = stg[g * G + u0 + u];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (u0 + u < len) num = __dadd_rn(num, v[u]);
        }
      } else if (variant == 1) {  // zero-padded, branch-free adds (x + 0.0 == x for x != -0)
        for (int u0 = 0; u0 < len; u0 += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (u0 + u < len) ? stg[g * G + u0 + u] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) num = __dadd_rn(num, v[u]);
        }
      } else if (variant == 2) {  // plain loop
        for (int u = 0; u < len; ++u) num = __dadd_rn(num, stg[g * G + u]);
      } else {  // conflict-free layout: lane g reads its own bank-staggered row
        for (int u0 = 0; u0 < len; u0 += 8) {
          double v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = (u0 + u < len) ? stg[(u0 + u) * 4 + g] : 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) num = __dadd_rn(num, v[u]);
        }
      }
    }
    __syncwarp();
  }
  long long t1 = clock64();
  if (park) asm volatile("bar.sync 1, %0;" ::"r"((int)blockDim.x) : "memory");
  if (tid == 0) { out[0] = t1 - t0; out[1] = (long long)num; }
}
int main() {
  long long* o; long long h[2];
  cudaMalloc(&o, 16);
  for (int park : {0, 1})
    for (int T : {32, 512})
      for (int variant = 0; variant < 4; ++variant)
        for (int len : {8, 13, 27}) {
          kchain<<<1, T>>>(o, len, variant, park);
          kchain<<<1, T>>>(o, len, variant, park);
          cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
          printf("park=%d T=%3d variant=%d len=%2d: %6.1f cycles/add\n", park, T, variant, len,
                 h[0] / (16.0 * len));
        }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
