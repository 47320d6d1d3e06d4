// Latency microbenchmarks of the primitives the resident sweep is built from (B200 sm_100a).
#include <cstdio>
#include <cstdint>
__global__ void kb(long long* out, const int* chase_g, int n_iter) {
  __shared__ int chase[1024];
  __shared__ double sd[1024];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += blockDim.x) { chase[i] = (i * 37 + 11) & 1023; sd[i] = 1.0 + i; }
  __syncthreads();
  long long t0, t1;
  // 1. dependent DADD chain (thread 0)
  if (tid == 0) {
    double x = sd[3];
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) x = __dadd_rn(x, 1.0000001);
    t1 = clock64();
    out[0] = (t1 - t0); out[15] = (long long)x;
    double y = sd[5];
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) y = __ddiv_rn(y, 1.0000001);
    t1 = clock64();
    out[1] = (t1 - t0); out[14] = (long long)y;
    int p = 0;
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) p = chase[p];
    t1 = clock64();
    out[2] = (t1 - t0); out[13] = p;
    p = 0;
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) p = __ldcg(&chase_g[p]);
    t1 = clock64();
    out[3] = (t1 - t0); out[12] = p;
    double z = sd[7];
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) z = __fma_rn(z, 1.0000001, 0.5);
    t1 = clock64();
    out[4] = (t1 - t0); out[11] = (long long)z;
  }
  __syncthreads();
  // 2. named barrier over first 128 threads
  if (tid < 128) {
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) asm volatile("bar.sync 1, 128;" ::: "memory");
    t1 = clock64();
    if (tid == 0) out[5] = t1 - t0;
  }
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < n_iter; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) out[6] = t1 - t0;
  int acc = 0;
  t0 = clock64();
  for (int i = 0; i < n_iter; ++i) acc += __syncthreads_or(i == tid);
  t1 = clock64();
  if (tid == 0) { out[7] = t1 - t0; out[10] = acc; }
  // 3. dependent DADD chain with DMUL operand from smem (the sweep's inner op)
  if (tid == 0) {
    double num = 0.0;
    int j = 0;
    t0 = clock64();
    for (int i = 0; i < n_iter; ++i) { num = __dadd_rn(num, __dmul_rn(3.0, sd[j])); j = (j + 7) & 1023; }
    t1 = clock64();
    out[8] = t1 - t0; out[9] = (long long)num;
  }
}
int main() {
  int* g; long long* o; long long h[16];
  cudaMalloc(&g, 4096 * 4); cudaMalloc(&o, 16 * 8);
  int hg[4096]; for (int i = 0; i < 4096; ++i) hg[i] = (i * 1237 + 11) & 4095;
  cudaMemcpy(g, hg, sizeof(hg), cudaMemcpyHostToDevice);
  const int N = 1000;
  for (int T : {128, 256, 512, 1024}) {
    kb<<<1, T>>>(o, g, N);  // warm
    kb<<<1, T>>>(o, g, N);
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("T=%4d cycles/op: dadd %.1f ddiv %.1f lds-chase %.1f l2-chase %.1f dfma %.1f bar128 %.1f syncthreads %.1f syncthreads_or %.1f dmul+dadd+lds %.1f\n",
           T, h[0] / (double)N, h[1] / (double)N, h[2] / (double)N, h[3] / (double)N, h[4] / (double)N,
           h[5] / (double)N, h[6] / (double)N, h[7] / (double)N, h[8] / (double)N);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
