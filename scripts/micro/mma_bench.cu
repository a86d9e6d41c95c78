// tcgen05 kind::i8 throughput microbenchmark: the K1 MMA mix (M=128, K=32, N=192 unsigned + N=32 signed,
// 2 M tiles x 2 K steps per 64-row tile), A from TMEM vs A from SMEM.
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
__device__ __forceinline__ uint32_t idesc_i8(int n, bool b_signed) {
  uint32_t d = 0;
  d |= 2u << 4; d |= 1u << 7; d |= (b_signed ? 1u : 0u) << 10;
  d |= static_cast<uint32_t>(n >> 3) << 17; d |= static_cast<uint32_t>(128 >> 4) << 24;
  return d;
}
template <int MODE>   // 0: A tmem, 192+32; 1: A smem, 192+32; 2: A tmem, single N=224 (unsigned); 3: A smem N=256
__global__ void __launch_bounds__(128, 1) mma_kernel(int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  uint8_t* A = sm;              // 256 rows x 64 K bytes
  uint8_t* B = sm + 16384;      // 256 x 64
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int chA = 256 / 8 * 128, chB = 224 / 8 * 128;
    for (int t = 0; t < tiles; ++t) {
      for (int ks = 0; ks < 2; ++ks)
        for (int tm = 0; tm < 2; ++tm) {
          const uint32_t acc = (t | ks) ? 1u : 0u;
          const uint32_t d = tmem + tm * 224;
          const uint32_t at = tmem + 448 + tm * 16 + ks * 8;
          const uint64_t ad = umma_desc(smem_u32(A) + 2 * ks * chA + tm * 16 * 128, chA, 128);
          if (MODE == 0 || MODE == 1) {
            const uint64_t bd0 = umma_desc(smem_u32(B) + 2 * ks * chB, chB, 128);
            const uint64_t bd1 = umma_desc(smem_u32(B) + 2 * ks * chB + (192 / 8) * 128, chB, 128);
            if (MODE == 0) {
              asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                           ::"r"(d), "r"(at), "l"(bd0), "r"(idesc_i8(192, false)), "r"(acc));
              asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                           ::"r"(d + 192), "r"(at), "l"(bd1), "r"(idesc_i8(32, true)), "r"(acc));
            } else {
              asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                           ::"r"(d), "l"(ad), "l"(bd0), "r"(idesc_i8(192, false)), "r"(acc));
              asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                           ::"r"(d + 192), "l"(ad), "l"(bd1), "r"(idesc_i8(32, true)), "r"(acc));
            }
          } else if (MODE == 2) {
            const uint64_t bd0 = umma_desc(smem_u32(B) + 2 * ks * chB, chB, 128);
            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(at), "l"(bd0), "r"(idesc_i8(224, false)), "r"(acc));
          } else {
            const int chB2 = 256 / 8 * 128;
            const uint64_t bd0 = umma_desc(smem_u32(B) + 2 * ks * chB2, chB2, 128);
            if (tm == 0)
              asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                           ::"r"(tmem), "l"(ad), "l"(bd0), "r"(idesc_i8(256, false)), "r"(acc));
          }
        }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[MODE] = (t1 - t0) / tiles;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
int main() {
  long long* out; cudaMallocManaged(&out, 8 * sizeof(long long));
  const int smem = 40960;
  cudaFuncSetAttribute(mma_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(mma_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_kernel<0><<<148, 128, smem>>>(3000, out);
  mma_kernel<1><<<148, 128, smem>>>(3000, out);
  mma_kernel<2><<<148, 128, smem>>>(3000, out);
  mma_kernel<3><<<148, 128, smem>>>(3000, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err=%s\ncycles per 64-row tile (ideal 448 @8192 MAC/clk):\n A tmem 192+32: %lld\n A smem 192+32: %lld\n A tmem N=224: %lld\n A smem N=256 (1 Mtile, ideal 256): %lld\n",
         cudaGetErrorString(e), out[0], out[1], out[2], out[3]);
  return 0;
}
