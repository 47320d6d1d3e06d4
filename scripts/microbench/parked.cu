// Does a lone working warp slow down while the rest of the block waits at __syncthreads?
// Also: smem ATOMS-with-return latency, and large dynamic smem.
#include <cstdio>
extern __shared__ int dyn[];
__global__ void k(long long* out, int park, int n, int use_dyn) {
  __shared__ int st[4096];
  int* chase = use_dyn ? dyn : st;
  const int tid = threadIdx.x;
  for (int i = tid; i < 4096; i += blockDim.x) chase[i] = (i * 37 + 11) & 4095;
  __syncthreads();
  if (tid >= 32) {
    if (park) __syncthreads();
    return;
  }
  long long t0 = clock64();
  int p = tid;
  for (int i = 0; i < n; ++i) p = chase[p];          // dependent LDS chain
  long long t1 = clock64();
  int q = tid;
  for (int i = 0; i < n; ++i) q = atomicAdd(&chase[q & 4095], 0) & 4095;  // dependent ATOMS
  long long t2 = clock64();
  double x = 1.0 + tid;
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, 1.0000001);
  long long t3 = clock64();
  if (park) __syncthreads();
  if (tid == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = p + q + (int)x; }
}
int main() {
  long long* o; long long h[4];
  cudaMalloc(&o, 32);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int dynb : {0, 1})
    for (int T : {32, 512})
      for (int park : {0, 1}) {
        size_t sm = dynb ? 200 * 1024 : 0;
        k<<<1, T, sm>>>(o, park, 1000, dynb); k<<<1, T, sm>>>(o, park, 1000, dynb);
        cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
        printf("dyn200KB=%d T=%3d park=%d: LDS %.1f  ATOMS-ret %.1f  DADD %.1f cycles\n", dynb, T, park,
               h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
