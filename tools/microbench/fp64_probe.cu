// FP64 / atomics / smem probes for the B200 design decisions in DESIGN.md.
// Not part of the product path: a one-off measurement tool run under gpurun.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__constant__ double cB[64];

// 8 independent DFMA chains per thread, register operands.
__global__ void dfma_reg(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// Same with the multiplier from __constant__ memory at compile-time offsets (c[][] operand).
__global__ void dfma_const(double* out, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, cB[u], x1); x1 = fma(x1, cB[u + 8], x2); x2 = fma(x2, cB[u + 16], x3); x3 = fma(x3, cB[u + 24], x4);
      x4 = fma(x4, cB[u + 32], x5); x5 = fma(x5, cB[u + 40], x6); x6 = fma(x6, cB[u + 48], x7); x7 = fma(x7, cB[u + 56], x0);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// DMMA m8n8k4: 4 independent accumulators per warp.
__global__ void dmma_884(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[2][0] + c[3][1];
}

// DMMA m16n8k16 (sm_90+ f64 shape): 8 A regs, 4 B regs, 4 C regs.
__global__ void dmma_16816(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[2][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 2; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[0][2] + c[1][3];
}

// red.global.add.f64: each thread adds into a contiguous window (element-like scatter).
__global__ void red_f64(double* y, long n, int per_thread, int stride) {
  long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
  for (int k = 0; k < per_thread; ++k) {
    long idx = ((t + (long)k * stride) * 7) % n;
    atomicAdd(&y[idx], 1.0);
  }
}

// streaming read + write (x -> y) double2
__global__ void copy_f64(const double2* __restrict__ x, double2* __restrict__ y, long n2) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) y[i] = x[i];
}

// smem LDS.64 throughput: each thread reads consecutive doubles (conflict-free).
__global__ void lds64(double* out, int iters) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int base = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int o = (base + u * 256 + i) & 4095;
      acc0 += s[o]; acc1 += s[(o + 32) & 4095]; acc2 += s[(o + 64) & 4095]; acc3 += s[(o + 96) & 4095];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

template <class F>
float timeit(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  int smem_optin = 0; CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"mem_gb\":%.1f}\n", prop.name, sms, l2,
         smem_optin, prop.totalGlobalMem / 1e9);
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.999 - i * 1e-4;
  CK(cudaMemcpyToSymbol(cB, h, sizeof(h)));
  double* out; CK(cudaMalloc(&out, 1 << 26));
  const int iters = 4096;
  for (int bs : {128, 256, 512}) {
    int grid = sms * (2048 / bs);
    float ms = timeit([&] { dfma_reg<<<grid, bs>>>(out, iters, 0.999, 1e-3); });
    double fl = 2.0 * 64 * iters * (double)grid * bs;
    printf("{\"probe\":\"dfma_reg\",\"block\":%d,\"tflops\":%.2f}\n", bs, fl / ms / 1e9);
    ms = timeit([&] { dfma_const<<<grid, bs>>>(out, iters); });
    printf("{\"probe\":\"dfma_const\",\"block\":%d,\"tflops\":%.2f}\n", bs, fl / ms / 1e9);
  }
  {
    int bs = 256, grid = sms * 8;
    float ms = timeit([&] { dmma_884<<<grid, bs>>>(out, iters); });
    double fl = 2.0 * 8 * 8 * 4 * 16.0 * iters * (double)grid * (bs / 32);
    printf("{\"probe\":\"dmma_m8n8k4\",\"tflops\":%.2f}\n", fl / ms / 1e9);
    ms = timeit([&] { dmma_16816<<<grid, bs>>>(out, iters); });
    fl = 2.0 * 16 * 8 * 16 * 2.0 * iters * (double)grid * (bs / 32);
    printf("{\"probe\":\"dmma_m16n8k16\",\"tflops\":%.2f}\n", fl / ms / 1e9);
  }
  {
    long n = 1L << 27;  // 1 GiB of doubles
    double *x, *y; CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8)); CK(cudaMemset(x, 0, n * 8));
    float ms = timeit([&] { copy_f64<<<sms * 16, 256>>>((double2*)x, (double2*)y, n / 2); });
    printf("{\"probe\":\"copy_f64\",\"gbs\":%.1f}\n", 2.0 * n * 8 / ms / 1e6);
    for (int stride : {1, 4096}) {
      int per = 16; long threads = n / per;
      ms = timeit([&] { red_f64<<<(int)(threads / 256), 256>>>(y, n, per, stride); });
      printf("{\"probe\":\"red_f64\",\"stride\":%d,\"gops\":%.1f}\n", stride, (double)threads * per / ms / 1e6);
    }
    CK(cudaFree(x)); CK(cudaFree(y));
  }
  {
    int bs = 256, grid = sms * 8;
    float ms = timeit([&] { lds64<<<grid, bs>>>(out, iters); });
    double bytes = 8.0 * 32 * iters * (double)grid * bs;
    printf("{\"probe\":\"lds64\",\"tbs\":%.2f,\"bytes_per_clk_per_sm_at_1965\":%.1f}\n", bytes / ms / 1e9,
           bytes / ms / 1e-3 / sms / 1.965e9);
  }
  return 0;
}
