// Cost of cross-CTA signalling inside a 2-CTA cluster (sm_100a): a warp of CTA 1 issues N
// operations to CTA 0, timed with clock64 on the issuing side.
//   MODE 0: mbarrier.arrive.shared::cluster (default .release.cta) on CTA 0's barrier
//   MODE 1: mbarrier.arrive.release.cluster.shared::cluster
//   MODE 2: st.async (4 bytes, complete_tx) into CTA 0
//   MODE 3: local mbarrier.arrive on CTA 1's own barrier (baseline)
//   MODE 4: STS (64 B per lane) + fence.proxy.async + remote arrive (the K1 slicer's publish)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) k(int n, long long* out) {
  __shared__ uint64_t bar;
  __shared__ uint32_t buf[4096];
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1 << 20));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t rbar, rbuf;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbar) : "r"(smem_u32(&bar)));
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbuf) : "r"(smem_u32(&buf[threadIdx.x])));
  long long t0 = clock64();
  if (rank == 1 && threadIdx.x < 32) {
    for (int i = 0; i < n; ++i) {
      if (MODE == 0) { if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory"); }
      if (MODE == 1) { if (threadIdx.x == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory"); }
      if (MODE == 2) { if (threadIdx.x == 0) asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(rbuf), "r"(i), "r"(rbar) : "memory"); }
      if (MODE == 3) { if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory"); }
      if (MODE == 4) {
        for (int j = 0; j < 16; ++j) buf[(threadIdx.x * 16 + j + i) & 4095] = i + j;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
      }
      __syncwarp();
    }
  }
  long long t1 = clock64();
  if (rank == 1 && threadIdx.x == 0 && blockIdx.x == 1) out[MODE] = (t1 - t0) / n;
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 64);
  const int n = 4096;
  k<0><<<2, 64>>>(n, out); k<1><<<2, 64>>>(n, out); k<2><<<2, 64>>>(n, out); k<3><<<2, 64>>>(n, out);
  k<4><<<2, 64>>>(n, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\ncycles per op (issuing warp): remote arrive %lld | remote arrive release.cluster %lld | st.async %lld | "
         "local arrive %lld | 16 STS + fence.proxy.async + remote arrive %lld\n",
         cudaGetErrorString(e), out[0], out[1], out[2], out[3], out[4]);
}
