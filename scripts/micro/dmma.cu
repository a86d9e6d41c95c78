#include <cstdio>
__global__ void dmma_k(int iters, double* out) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void dfma_k(int iters, double* out) {
  double c[16] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) c[k] = fma(a, b, c[k]);
  }
  double s = 0; for (int k = 0; k < 16; ++k) s += c[k];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; float ms;
  dmma_k<<<148 * 4, 256>>>(100, o); dfma_k<<<148 * 4, 256>>>(100, o);
  cudaEventRecord(e0); dmma_k<<<148 * 4, 256>>>(iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 148 * 4 * 8 * (double)iters * 8 * 256;   // per warp per mma 256 FMA
  printf("DMMA: %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
  cudaEventRecord(e0); dfma_k<<<148 * 4, 256>>>(iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 148 * 4 * 256 * (double)iters * 16;
  printf("DFMA: %.2f TFLOP/s\n", fl / (ms * 1e-3) / 1e12);
  return 0;
}
