// Probe 2: DFMA with a __constant__ operand in independent chains, and a
// "fiber contraction" microkernel (n inputs in registers, q outputs, constant-bank
// coefficients) = the inner loop shape of the apply kernel.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
__constant__ double cB[128];

__global__ void dfma_const_indep(double* out, int iters, double b) {
  double x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = threadIdx.x + u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = fma(x[u], cB[u * 8 + j], b);
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += x[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// out[a] = sum_i C[a][i] in[i], N=7 inputs, Q=8 outputs, repeated; inputs perturbed each iter
template <int N, int Q>
__global__ void fiber(double* out, int iters) {
  double in[N];
#pragma unroll
  for (int i = 0; i < N; ++i) in[i] = threadIdx.x * 1e-3 + i;
  double acc[Q];
#pragma unroll
  for (int a = 0; a < Q; ++a) acc[a] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int a = 0; a < Q; ++a) {
      double s = acc[a];
#pragma unroll
      for (int i = 0; i < N; ++i) s = fma(cB[a * N + i], in[i], s);
      acc[a] = s;
    }
#pragma unroll
    for (int i = 0; i < N; ++i) in[i] = fma(in[i], 0.999, acc[i % Q] * 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int a = 0; a < Q; ++a) s += acc[a];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class F> float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) { CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms; }
  CK(cudaGetLastError()); return best;
}

int main() {
  int sms = 148;
  double h[128]; for (int i = 0; i < 128; ++i) h[i] = 0.999 - i * 1e-4;
  CK(cudaMemcpyToSymbol(cB, h, sizeof(h)));
  double* out; CK(cudaMalloc(&out, 1 << 26));
  const int iters = 2048;
  for (int bs : {128, 256}) for (int occ : {2, 4, 8}) {
    int grid = sms * occ * (256 / bs);
    float ms = timeit([&] { dfma_const_indep<<<grid, bs>>>(out, iters, 1e-3); });
    double fl = 2.0 * 64 * iters * (double)grid * bs;
    printf("{\"probe\":\"dfma_const_indep\",\"block\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f}\n", bs, occ * 8, fl / ms / 1e9);
  }
  for (int occ : {1, 2, 4, 8}) {
    int bs = 256, grid = sms * occ;
    float ms = timeit([&] { fiber<7, 8><<<grid, bs>>>(out, iters); });
    double fl = 2.0 * (56 + 7) * iters * (double)grid * bs;
    printf("{\"probe\":\"fiber_7x8\",\"warps_per_sm\":%d,\"tflops\":%.2f}\n", occ * 8, fl / ms / 1e9);
  }
  return 0;
}
