// Can the FP64 tensor path (DMMA, mma.sync m16n8k4 f64) and the FP64 FMA pipe (DFMA) run at the same
// time on B200?  One kernel, 8 warps per CTA: warps [0, nd) issue independent DMMA chains, the
// others independent DFMA chains; the same per-warp work in "DMMA only", "DFMA only" and "mixed"
// launches.  If the two share one datapath the mixed time is the sum; if not, the max.
#include <cstdio>
#include <cuda_runtime.h>

#define MMA_K4(c, a, b)                                                                                 \
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]))

__global__ void mixed(double* out, int iters, int nd_warps, int nf_warps) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w < nd_warps) {
    double a[2] = {1e-3 * threadIdx.x, 2e-3}, b[1] = {1.0 - 1e-4 * threadIdx.x}, c[8][4];
    for (int u = 0; u < 8; ++u) c[u][0] = c[u][1] = c[u][2] = c[u][3] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int u = 0; u < 8; ++u) MMA_K4(c[u], a, b);
      a[0] += 1e-9;
    }
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  } else if (w < nd_warps + nf_warps) {
    double x[16];
    for (int u = 0; u < 16; ++u) x[u] = threadIdx.x + u;
    const double m = 0.999999, k = 1e-7;
    // per iteration 16 chains x 16 DFMA = 256 DFMA per thread = 8192 per warp = the MACs of
    // 16 m16n8k4 DMMAs (512 MAC each) -> 2x the DMMA warp's 8 per iteration: run half the iterations
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = fma(x[u], m, k);
    }
    for (int u = 0; u < 16; ++u) s += x[u];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 4 * 256);
  const int iters = 4096, grid = 148 * 2, bs = 256;   // 2 CTAs x 8 warps per SM
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int cases[3][2] = {{4, 0}, {0, 4}, {4, 4}};
  const char* names[3] = {"dmma_only(4 warps)", "dfma_only(4 warps)", "mixed(4+4 warps)"};
  for (int c = 0; c < 3; ++c) {
    mixed<<<grid, bs>>>(out, iters, cases[c][0], cases[c][1]);
    cudaEventRecord(e0);
    mixed<<<grid, bs>>>(out, iters, cases[c][0], cases[c][1]);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // MACs: DMMA warp 8 x 512 per iteration; DFMA warp 8 x 16 x 32 = 4096 per iteration
    const double macs = (double)grid * iters * (cases[c][0] * 8.0 * 512 + cases[c][1] * 4096.0);
    printf("{\"case\":\"%s\",\"ms\":%.3f,\"fp64_tflops\":%.2f,\"err\":\"%s\"}\n", names[c], ms,
           2.0 * macs / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
