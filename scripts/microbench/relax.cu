// Cost of one relaxation round (K8 sweep schedule): P threads, each: e (~7) dependent-free
// smem loads through a u16 list, max, store, then an OR barrier over P threads.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ int bar_or(int id, int n, int pred) {
  int r;
  asm volatile("{\n .reg .pred p, q;\n setp.ne.s32 p, %3, 0;\n bar.red.or.pred q, %1, %2, p;\n"
               " selp.s32 %0, 1, 0, q;\n}" : "=r"(r) : "r"(id), "r"(n), "r"(pred) : "memory");
  return r;
}
template <int BIGSMEM>
__global__ void k(int m, int rounds, int PW, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  int* lev = (int*)sm;
  int* nbe = lev + 1024;
  uint16_t* lst = (uint16_t*)(nbe + 1024);
  const int tid = threadIdx.x, T = blockDim.x;
  for (int i = tid; i < 1024; i += T) { lev[i] = i & 7; nbe[i] = 7; }
  for (int i = tid; i < 1024 * 28; i += T) lst[i] = (uint16_t)((i * 2654435761u >> 7) & 1023);
  __syncthreads();
  const int P = PW * 32;
  long long t0 = clock64();
  if ((tid >> 5) < PW) {
    for (int r = 0; r < rounds; ++r) {
      int changed = 0;
      for (int i = tid; i < m; i += P) {
        const int e = nbe[i];
        const uint16_t* li = lst + i * 28;
        int L = 0;
#pragma unroll 4
        for (int t = 0; t < e; ++t) L = max(L, lev[li[t]] + 1);
        if (L != lev[i]) { lev[i] = L & 7; changed = 1; }
      }
      bar_or(3, P, changed | (r < rounds));
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (tid == 0) out[0] = t1 - t0;
}
int main() {
  long long* o; cudaMalloc(&o, 8);
  size_t big = 200 * 1024, small = 1024 * 8 + 1024 * 28 * 2;
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)big);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)small);
  for (int m : {64, 433}) for (int PW : {2, 14}) {
    if (PW * 32 < m && PW == 2) {}
    long long h;
    k<0><<<1, 512, small>>>(m, 50, PW, o); k<0><<<1, 512, small>>>(m, 50, PW, o);
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("m=%3d PW=%2d small smem: %7.1f cycles/round\n", m, PW, h / 50.0);
    k<1><<<1, 512, big>>>(m, 50, PW, o); k<1><<<1, 512, big>>>(m, 50, PW, o);
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("m=%3d PW=%2d 200KB smem: %7.1f cycles/round  %s\n", m, PW, h / 50.0, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
