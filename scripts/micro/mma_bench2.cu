// tcgen05 kind::i8 throughput with the CTA pair (cta_group::2, M = 256): the K1 MMA mix per 64-row
// tile (2 M tiles x 2 K steps x {N = 192 unsigned + N = 32 signed}), A from TMEM, B from SMEM
// (N split across the pair).  MODE 0: one commit at the end; 1: two commits per tile (as K1);
// 2: single N = 224 MMA per (M tile, K step); 3: cta_group::1 (M = 128) with per-tile commits.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}
__device__ __forceinline__ uint32_t idesc_i8(int m, int n, bool b_signed) {
  uint32_t d = 0;
  d |= 2u << 4; d |= 1u << 7; d |= (b_signed ? 1u : 0u) << 10;
  d |= static_cast<uint32_t>(n >> 3) << 17; d |= static_cast<uint32_t>(m >> 4) << 24;
  return d;
}
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_kernel(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[3];
  __shared__ uint32_t tbase;
  constexpr bool G2 = MODE != 3;
  uint8_t* B = sm;      // 112 rows (per CTA) x 64 K bytes
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    if (G2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (threadIdx.x == 0)
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(1));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  const int MM = G2 ? 256 : 128;
  const int NU = G2 ? 192 : 192, NS = 32;
  const int rows = G2 ? 112 : 224;          // B rows per CTA
  const int chB = rows / 8 * 128;
  if (threadIdx.x < 32 && (rank == 0 || !G2)) {
    for (int t = 0; t < tiles; ++t) {
      for (int ks = 0; ks < 2; ++ks)
        for (int tm = 0; tm < 2; ++tm) {
          const uint32_t acc = (t | ks) ? 1u : 0u;
          const uint32_t d = tmem + tm * 224;
          const uint32_t at = tmem + 448 + (t & 1) * 32 + tm * 16 + ks * 8;
          const uint32_t bst = smem_u32(B) + (MODE == 4 ? (t & 7) * 7168 : 0);
          const uint64_t bd0 = umma_desc(bst + 2 * ks * chB, chB, 128);
          const uint64_t bd1 = umma_desc(bst + 2 * ks * chB + ((G2 ? 96 : 192) / 8) * 128, chB, 128);
          if (MODE == 2) {
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(at), "l"(bd0), "r"(idesc_i8(MM, 224, false)), "r"(acc));
          } else if (G2) {
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(at), "l"(bd0), "r"(idesc_i8(MM, NU, false)), "r"(acc));
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d + NU), "r"(at), "l"(bd1), "r"(idesc_i8(MM, NS, true)), "r"(acc));
          } else {
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(at), "l"(bd0), "r"(idesc_i8(MM, NU, false)), "r"(acc));
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d + NU), "r"(at), "l"(bd1), "r"(idesc_i8(MM, NS, true)), "r"(acc));
          }
        }
      if (MODE == 1 || MODE == 4) {
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}"
                     ::"r"(smem_u32(&bar[1])), "h"((uint16_t)3) : "memory");
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}"
                     ::"r"(smem_u32(&bar[2])), "h"((uint16_t)3) : "memory");
      } else if (MODE == 3) {
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}"
                     ::"r"(smem_u32(&bar[1])) : "memory");
        asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}"
                     ::"r"(smem_u32(&bar[2])) : "memory");
      }
    }
    if (G2)
      asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}"
                   ::"r"(smem_u32(&bar[0])), "h"((uint16_t)3) : "memory");
    else
      asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}"
                   ::"r"(smem_u32(&bar[0])) : "memory");
  }
  if (threadIdx.x == 0)
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar[0])) : "memory");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[MODE] = (t1 - t0) / tiles;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (threadIdx.x < 32) {
    if (G2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 8 * sizeof(long long));
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(mma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_kernel<4><<<148, 128, smem>>>(3000, out);
  mma_kernel<0><<<148, 128, smem>>>(3000, out);
  mma_kernel<1><<<148, 128, smem>>>(3000, out);
  mma_kernel<2><<<148, 128, smem>>>(3000, out);
  mma_kernel<3><<<148, 128, smem>>>(3000, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\ncycles per 64-row tile (ideal 448):\n 2SM 192+32 commit at end: %lld\n 2SM 192+32 2 commits/tile: %lld\n"
         " 2SM N=224: %lld\n 1SM 192+32 2 commits/tile: %lld\n 2SM rotating 8 B stages: %lld\n", cudaGetErrorString(e), out[0], out[1], out[2], out[3], out[4]);
  return 0;
}
