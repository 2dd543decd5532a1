// Warp LU variants on sm_100a: dependent-chain cycles (clock64, one warp) and bit-equality with the
// scalar restatement dev_lu_solve (kernels.cpp:95-154) over random, ill-scaled, pivoting-heavy and
// singular systems. Developer tool: nvcc -I paper_1604_06043_b200/csrc ... tools/ubench/lu.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kcommon.cuh"

using namespace mstab_b200;
namespace mstab_b200 {
int g_num_sms = 148;
std::mutex g_occ_mu;
std::unordered_map<const void*, int> g_occ;
}

template <int S, int VARIANT>
__global__ void k_lu(const double* m, const double* rhs, double* xout, int* okout, long long* cyc, int nsys) {
  __shared__ double lu[S * S], vin[S], vout[S];
  long long total = 0;
  for (int sys = 0; sys < nsys; ++sys) {
    for (int i = threadIdx.x; i < S * S; i += 32) lu[i] = m[sys * S * S + i];
    if (threadIdx.x < S) {
      vin[threadIdx.x] = rhs[sys * S + threadIdx.x];
      vout[threadIdx.x] = -777.0;
    }
    __syncwarp();
    const long long t0 = clock64();
    bool ok;
    if (VARIANT == 0) {
      ok = false;
      if (threadIdx.x == 0) ok = dev_lu_solve(S, lu, vin, vout);
      ok = __shfl_sync(0xffffffffu, ok, 0);
    } else if (VARIANT == 1) {
      ok = warp_lu_impl<S, true>(S, lu, vin, vout);
    } else {
      ok = warp_lu_fixed<S>(lu, vin, vout);
    }
    __syncwarp();
    if (sys % 8 == 0) total += clock64() - t0;  // the plain random (nonsingular) systems
    if (threadIdx.x < S) xout[sys * S + threadIdx.x] = ok ? vout[threadIdx.x] : 0.0;
    if (threadIdx.x == 0) okout[sys] = ok ? 1 : 0;
    __syncwarp();
  }
  if (threadIdx.x == 0) *cyc = total / ((nsys + 7) / 8);
}

static double urand() { return (double)rand() / RAND_MAX * 2.0 - 1.0; }

template <int S>
void run() {
  const int nsys = 2000;
  std::vector<double> m((size_t)nsys * S * S), rhs((size_t)nsys * S);
  srand(1234 + S);
  for (int sys = 0; sys < nsys; ++sys) {
    double* a = &m[(size_t)sys * S * S];
    for (int i = 0; i < S * S; ++i) a[i] = urand();
    const int kind = sys % 8;
    if (kind == 1)  // badly scaled rows
      for (int i = 0; i < S; ++i) { const double sc = std::ldexp(1.0, (rand() % 40) - 20); for (int j = 0; j < S; ++j) a[i + j * S] *= sc; }
    if (kind == 2 && S > 1)  // exactly singular: two equal columns
      for (int i = 0; i < S; ++i) a[i + 1 * S] = a[i + 0 * S];
    if (kind == 3)  // ties in the pivot search, zeros (skipped eliminations)
      for (int i = 0; i < S * S; ++i) a[i] = (double)((rand() % 5) - 2);
    if (kind == 4) std::memset(a, 0, sizeof(double) * S * S);  // zero matrix
    if (kind == 5)  // nearly singular
      for (int i = 0; i < S; ++i) a[i + (S - 1) * S] = a[i] * (1.0 + 1e-15 * urand());
    for (int i = 0; i < S; ++i) rhs[(size_t)sys * S + i] = kind == 6 ? 0.0 : urand();
  }
  double *dm, *dr, *dx[3];
  int* dok[3];
  long long* dc;
  cudaMalloc(&dm, m.size() * 8);
  cudaMalloc(&dr, rhs.size() * 8);
  cudaMallocManaged(&dc, 3 * 8);
  cudaMemcpy(dm, m.data(), m.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rhs.data(), rhs.size() * 8, cudaMemcpyHostToDevice);
  for (int v = 0; v < 3; ++v) {
    cudaMalloc(&dx[v], rhs.size() * 8);
    cudaMalloc(&dok[v], nsys * 4);
  }
  for (int rep = 0; rep < 2; ++rep) {
    k_lu<S, 0><<<1, 32>>>(dm, dr, dx[0], dok[0], dc + 0, nsys);
    k_lu<S, 1><<<1, 32>>>(dm, dr, dx[1], dok[1], dc + 1, nsys);
    k_lu<S, 2><<<1, 32>>>(dm, dr, dx[2], dok[2], dc + 2, nsys);
    cudaDeviceSynchronize();
  }
  std::vector<double> x[3];
  std::vector<int> ok[3];
  for (int v = 0; v < 3; ++v) {
    x[v].resize(rhs.size());
    ok[v].resize(nsys);
    cudaMemcpy(x[v].data(), dx[v], rhs.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(ok[v].data(), dok[v], nsys * 4, cudaMemcpyDeviceToHost);
  }
  int bad1 = 0, bad2 = 0, nsing = 0;
  for (int sys = 0; sys < nsys; ++sys) {
    nsing += !ok[0][sys];
    bool e1 = ok[1][sys] == ok[0][sys], e2 = ok[2][sys] == ok[0][sys];
    if (ok[0][sys]) {
      e1 = e1 && !std::memcmp(&x[1][(size_t)sys * S], &x[0][(size_t)sys * S], 8 * S);
      e2 = e2 && !std::memcmp(&x[2][(size_t)sys * S], &x[0][(size_t)sys * S], 8 * S);
    }
    bad1 += !e1;
    bad2 += !e2;
  }
  printf("S=%2d  cycles/solve: scalar %6lld  warp_lu_impl %6lld  warp_lu_fixed %6lld   mismatches vs scalar: impl %d fixed %d of %d (%d singular)  %s\n",
         S, dc[0], dc[1], dc[2], bad1, bad2, nsys, nsing, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<1>();
  run<2>();
  run<3>();
  run<4>();
  run<6>();
  run<8>();
  run<12>();
  run<16>();
  return 0;
}
