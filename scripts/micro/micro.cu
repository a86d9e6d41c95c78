// Microbenchmarks for the post-pass design: cluster barrier, fp64 dependent-chain latency,
// fp64 divide latency, DSMEM store + barrier.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(16, 1, 1) clusync_kernel(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}
__global__ void __cluster_dims__(16, 1, 1) clusync_split_kernel(int iters, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (t1 - t0) / iters;
}
__global__ void dchain_kernel(int iters, double a, double* sink, long long* out) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, 1e-7);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[2] = (t1 - t0) / iters; sink[0] = x; }
}
__global__ void ddiv_kernel(int iters, double a, double* sink, long long* out) {
  double x = 1.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = a / x + 0.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[3] = (t1 - t0) / iters; sink[1] = x; }
}
__global__ void __cluster_dims__(16, 1, 1) dsmem_kernel(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[16 * 32];
  const int c = cl.block_rank();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    for (int t = threadIdx.x; t < 32 * 16; t += blockDim.x) {
      const int q = t / 32, j = t % 32;
      double* dst = cl.map_shared_rank(buf, q);
      dst[c * 32 + j] = i + j;
    }
    cl.sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && c == 0) out[4] = (t1 - t0) / iters;
}
int main() {
  long long* out; double* sink;
  cudaMallocManaged(&out, 8 * sizeof(long long)); cudaMallocManaged(&sink, 8 * sizeof(double));
  cudaFuncSetAttribute(clusync_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(clusync_split_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(dsmem_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  clusync_kernel<<<16, 256>>>(1000, out);
  clusync_split_kernel<<<16, 256>>>(1000, out);
  dchain_kernel<<<1, 32>>>(10000, 0.999, sink, out);
  ddiv_kernel<<<1, 32>>>(10000, 0.7, sink, out);
  dsmem_kernel<<<16, 256>>>(1000, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\ncluster.sync (16 CTAs x 256 thr): %lld cycles\nsplit arrive/wait: %lld cycles\n"
         "dependent DFMA: %lld cycles\ndependent DDIV+add: %lld cycles\nDSMEM 4KB all-to-all + cluster.sync: %lld cycles\n",
         cudaGetErrorString(e), out[0], out[1], out[2], out[3], out[4]);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); clusync_kernel<<<16, 256>>>(10000, out); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); printf("10000 cluster.sync: %.3f ms -> %.3f us each\n", ms, ms * 1e3 / 10000);
  return 0;
}
