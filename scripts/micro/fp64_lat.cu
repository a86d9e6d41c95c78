// fp64 dependent-chain latency on sm_100a (DFMA / DADD / DMUL), one warp, clock64.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = __fma_rn(x, b, a);
    x = __fma_rn(x, b, a);
    x = __fma_rn(x, b, a);
    x = __fma_rn(x, b, a);
  }
  long long t1 = clock64();
  double y = a;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    y = __dadd_rn(y, b);
    y = __dadd_rn(y, b);
    y = __dadd_rn(y, b);
    y = __dadd_rn(y, b);
  }
  long long t2 = clock64();
  out[threadIdx.x] = x + y;
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 4096; cyc[1] = (t2 - t1) / 4096; }
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 1024 * 8); cudaMallocManaged(&c, 16);
  lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  printf("DFMA dependent latency %lld cycles, DADD %lld cycles\n", c[0], c[1]);
}
