// Verify the assumed register<->matrix mapping of mma.sync f64 m16n8k4 / m16n8k8 and time
// m16n8k4.  g = lane >> 2, t = lane & 3.
//   m16n8k4: A a0=A[g][t] a1=A[g+8][t]; B b0=B[t][g]; C c0=C[g][2t] c1=C[g][2t+1] c2=C[g+8][2t] c3=C[g+8][2t+1]
//   m16n8k8: A a0=A[g][t] a1=A[g+8][t] a2=A[g][t+4] a3=A[g+8][t+4]; B b0=B[t][g] b1=B[t+4][g]; C as above
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k4(const double* A, const double* B, double* C) {  // A 16x4, B 4x8, C 16x8
  int l = threadIdx.x, g = l >> 2, t = l & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t], b0 = B[t * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
  C[g * 8 + 2 * t] = c0; C[g * 8 + 2 * t + 1] = c1; C[(g + 8) * 8 + 2 * t] = c2; C[(g + 8) * 8 + 2 * t + 1] = c3;
}

__global__ void k8(const double* A, const double* B, double* C) {  // A 16x8, B 8x8
  int l = threadIdx.x, g = l >> 2, t = l & 3;
  double a0 = A[g * 8 + t], a1 = A[(g + 8) * 8 + t], a2 = A[g * 8 + t + 4], a3 = A[(g + 8) * 8 + t + 4];
  double b0 = B[t * 8 + g], b1 = B[(t + 4) * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  C[g * 8 + 2 * t] = c0; C[g * 8 + 2 * t + 1] = c1; C[(g + 8) * 8 + 2 * t] = c2; C[(g + 8) * 8 + 2 * t + 1] = c3;
}

__global__ void k4_rate(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = 1 - a0;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0][0] + c[1][1] + c[2][2] + c[3][3];
}

int main() {
  double hA[128], hB[64], hC[128], ref[128];
  for (int K : {4, 8}) {
    for (int i = 0; i < 16 * K; ++i) hA[i] = 1.0 + i * 0.37 + (i % 5) * 0.011;
    for (int i = 0; i < K * 8; ++i) hB[i] = -2.0 + i * 0.13 + (i % 3) * 0.007;
    for (int r = 0; r < 16; ++r)
      for (int n = 0; n < 8; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += hA[r * K + k] * hB[k * 8 + n];
        ref[r * 8 + n] = s;
      }
    double *dA, *dB, *dC;
    cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dC, sizeof(hC));
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    if (K == 4) k4<<<1, 32>>>(dA, dB, dC); else k8<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, sizeof(hC), cudaMemcpyDeviceToHost);
    double err = 0;
    for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hC[i] - ref[i]) / (1 + fabs(ref[i])));
    printf("{\"probe\":\"layout_m16n8k%d\",\"max_rel_err\":%.3e,\"ok\":%s}\n", K, err, err < 1e-13 ? "true" : "false");
  }
  double* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int grid = 148 * 8, iters = 4096;
  k4_rate<<<grid, 256>>>(out, iters);
  cudaEventRecord(a); k4_rate<<<grid, 256>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\":\"dmma_m16n8k4\",\"tflops\":%.2f}\n", 2.0 * 16 * 8 * 4 * 4.0 * iters * grid * 8 / ms / 1e9);
  return 0;
}
