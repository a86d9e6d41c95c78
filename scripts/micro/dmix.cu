#include <cstdio>
// warps < ndm: DMMA loop; others: DFMA loop.  Measures combined fp64 throughput.
__global__ void mix_k(int iters, int ndm, double* out) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w < ndm) {
    double c[8][2] = {};
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};" : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  } else {
    double c[16] = {};
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) c[k] = fma(a, b, c[k]);
    }
    for (int k = 0; k < 16; ++k) s += c[k];
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000, warps = 16;
  for (int ndm = 0; ndm <= warps; ndm += 4) {
    mix_k<<<148, 32 * warps>>>(10, ndm, o);
    cudaEventRecord(e0); mix_k<<<148, 32 * warps>>>(iters, ndm, o); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    // DMMA warp: iters * 8 mma * 512 flop; DFMA warp: iters*8 * 16 fma * 32 lanes * 2 flop = iters*8*1024
    double fl = 148.0 * (ndm * (double)iters * 8 * 512 + (warps - ndm) * (double)iters * 8 * 16 * 32 * 2);
    printf("dmma warps %2d / %d: %.2f TFLOP/s  (%.3f ms)\n", ndm, warps, fl / (ms * 1e-3) / 1e12, ms);
  }
  return 0;
}
