#include <cstdio>
template <int NACC>
__global__ void dmma_k(int iters, double* out) {
  double c[NACC][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int k = 0; k < NACC; ++k) s += c[k][0] + c[k][1];
  if (s == 1.2345) out[0] = s;
}
template <int NACC>
void run(int ctas_per_sm, int warps, double* o) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000; float ms;
  dmma_k<NACC><<<148 * ctas_per_sm, 32 * warps>>>(10, o);
  cudaEventRecord(e0); dmma_k<NACC><<<148 * ctas_per_sm, 32 * warps>>>(iters, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 148 * ctas_per_sm * warps * (double)iters * NACC * 256;
  printf("acc %2d  warps/SM %2d: %.2f TFLOP/s\n", NACC, ctas_per_sm * warps, fl / (ms * 1e-3) / 1e12);
}
int main() {
  double* o; cudaMalloc(&o, 8);
  run<8>(1, 8, o); run<16>(1, 8, o); run<32>(1, 8, o);
  run<8>(1, 16, o); run<16>(1, 16, o);
  run<8>(4, 8, o); run<16>(2, 8, o);
  return 0;
}
