// Dependent-chain latencies on sm_100a (cycles per op), single warp: DADD, DMUL, DFMA, fp64 division,
// fp64 reciprocal, 64-bit shuffle, shared-memory load->add, L2 load (ld.cg) round trip.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a0, double b0, const double* g) {
  __shared__ double sm[64];
  sm[threadIdx.x] = a0 + threadIdx.x;
  __syncwarp();
  double a = a0, b = b0;
  long long t0, t1;
  int slot = 0;
#define TIME(N, BODY)                                   \
  t0 = clock64();                                       \
  _Pragma("unroll 1") for (int i = 0; i < N / 8; ++i) { \
    BODY BODY BODY BODY BODY BODY BODY BODY             \
  }                                                     \
  t1 = clock64();                                       \
  if (threadIdx.x == 0) cyc[slot] = (t1 - t0) / N;      \
  ++slot;
  TIME(256, a = a + b;)
  TIME(256, a = a * b;)
  TIME(256, a = fma(a, b, b);)
  TIME(64, a = b / a;)
  TIME(64, a = 1.0 / a;)
  TIME(256, a = __shfl_sync(0xffffffffu, a, 1);)
  TIME(256, a = a + sm[((int)a) & 31];)
  TIME(64, a = a + __ldcg(g + (((int)a) & 31));)
  out[threadIdx.x] = a;
}
int main() {
  double *out, *g;
  long long* cyc;
  cudaMalloc(&out, 256);
  cudaMalloc(&g, 1024);
  cudaMemset(g, 0, 1024);
  cudaMallocManaged(&cyc, 64);
  for (int r = 0; r < 2; ++r) {
    k<<<1, 32>>>(out, cyc, 1.000001, 0.9999999, g);
    cudaDeviceSynchronize();
  }
  const char* names[] = {"dadd", "dmul", "dfma", "ddiv", "drcp", "shfl64", "lds+dadd", "ldcg+dadd"};
  for (int i = 0; i < 8; ++i) printf("%-10s %lld cycles\n", names[i], cyc[i]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
