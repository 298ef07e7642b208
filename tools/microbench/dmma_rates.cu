// DMMA throughput by shape on B200, same methodology for each: NCH independent accumulator
// chains per warp, operands varied per iteration so nothing is loop-invariant, result checked.
#include <cstdio>
#include <cuda_runtime.h>

#define MMA_K4(c, a, b)                                                                                 \
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]))
#define MMA_K8(c, a, b)                                                                                 \
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]))
#define MMA_K16(c, a, b)                                                                                \
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n" \
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]))
#define MMA_884(c, a, b)                                                                                \
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"           \
               : "+d"(c[0]), "+d"(c[1]) : "d"(a[0]), "d"(b[0]))

template <int SHAPE, int NCH>
__global__ void rate(double* out, int iters) {
  double a[8], b[4], c[NCH][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1e-3 * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - 1e-4 * (threadIdx.x + i);
#pragma unroll
  for (int u = 0; u < NCH; ++u)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[u][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < NCH; ++u) {
      if (SHAPE == 4) MMA_K4(c[u], a, b);
      if (SHAPE == 8) MMA_K8(c[u], a, b);
      if (SHAPE == 16) MMA_K16(c[u], a, b);
      if (SHAPE == 884) MMA_884(c[u], a, b);
    }
    a[0] += 1e-9;  // loop-carried operand change
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < NCH; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int SHAPE, int NCH>
void run(double* out, int warps_per_sm) {
  const int iters = 2048, bs = 128, grid = 148 * warps_per_sm / 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  rate<SHAPE, NCH><<<grid, bs>>>(out, iters);
  cudaEventRecord(e0);
  rate<SHAPE, NCH><<<grid, bs>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double macs = (SHAPE == 884 ? 8.0 * 8 * 4 : 16.0 * 8 * (SHAPE == 884 ? 4 : SHAPE));
  double fl = 2.0 * macs * NCH * iters * (double)grid * (bs / 32);
  printf("{\"shape\":%d,\"chains\":%d,\"warps_per_sm\":%d,\"tflops\":%.2f,\"err\":\"%s\"}\n", SHAPE, NCH,
         warps_per_sm, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 26);
  for (int w : {4, 8, 16}) {
    run<884, 4>(out, w);
    run<4, 4>(out, w);
    run<4, 8>(out, w);
    run<8, 4>(out, w);
    run<16, 4>(out, w);
  }
  return 0;
}
