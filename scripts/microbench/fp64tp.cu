// FP64 issue/latency on one SMSP: K independent DADD chains per thread, one warp with `act`
// active lanes, plus the same with smem-fed operands.  Cycles per DADD warp-instruction.
#include <cstdio>
template <int K>
__global__ void kch(double* out, long long* cyc, int n, int act, int mode) {
  __shared__ double sv[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sv[i] = 1e-3 * (i + 1);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  if ((int)threadIdx.x >= act) return;
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x + k;
  const double a = 1.0000001;
  int j = threadIdx.x * 3;
  long long t0 = clock64();
  if (mode == 0) {
    for (int i = 0; i < n; ++i)
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = __dadd_rn(x[k], a);
  } else {  // operand from smem (independent of the chain)
    for (int i = 0; i < n; ++i) {
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = __dadd_rn(x[k], sv[(j + k * 7) & 1023]);
      j += 5;
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int K>
void run(double* o, long long* c, int mode) {
  for (int act : {1, 32}) {
    long long h;
    kch<K><<<1, 32>>>(o, c, 1000, act, mode);
    kch<K><<<1, 32>>>(o, c, 1000, act, mode);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("mode %d K=%d act=%2d: %6.2f cycles per DADD instr, %6.2f per chain step\n", mode, K, act,
           h / (1000.0 * K), h / 1000.0);
  }
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 8);
  for (int mode : {0, 1}) {
    run<1>(o, c, mode); run<2>(o, c, mode); run<3>(o, c, mode); run<4>(o, c, mode); run<8>(o, c, mode);
  }
  return 0;
}
