// Does a running tcgen05 kind::i8 MMA stream slow down DFMA / integer ALU work on the same SM?
// Warp 0 issues the K1 MMA mix (cta_group::1, M = 128, N = 192 + 32, A from TMEM) for `tiles`
// tiles (MODE 1) or nothing (MODE 0); warps 1..8 run independent DFMA chains (KIND 0) or
// LOP3/PRMT chains (KIND 1) for a fixed count.  Prints the cycles the side warps took.
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
template <int MODE, int KIND>
__global__ void __launch_bounds__(288, 1) k(int tiles, int iters, long long* out, double* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (MODE == 1) {
      const int chB = 224 / 8 * 128;
      for (int t = 0; t < tiles; ++t)
        for (int ks = 0; ks < 2; ++ks)
          for (int tm = 0; tm < 2; ++tm) {
            const uint32_t acc = (t | ks) ? 1u : 0u;
            const uint32_t d = tmem + tm * 224;
            const uint32_t at = tmem + 448 + (t & 1) * 32 + tm * 16 + ks * 8;
            const uint64_t bd0 = umma_desc(smem_u32(sm) + 2 * ks * chB, chB, 128);
            const uint64_t bd1 = umma_desc(smem_u32(sm) + 2 * ks * chB + 24 * 128, chB, 128);
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d), "r"(at), "l"(bd0), "r"(idesc_i8(192, false)), "r"(acc));
            asm volatile("{.reg .pred p, e; elect.sync _|e, 0xffffffff; setp.ne.b32 p, %4, 0; @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                         ::"r"(d + 192), "r"(at), "l"(bd1), "r"(idesc_i8(32, true)), "r"(acc));
          }
      asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}"
                   ::"r"(smem_u32(&bar)) : "memory");
    }
  } else {
    long long t0 = clock64();
    if (KIND == 0) {
      double a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fma_rn(a[i], 1.0000001, 0.5);
      double s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += a[i];
      sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else if (KIND == 2) {
      float a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fmaf_rn(a[i], 1.0000001f, 0.5f);
      float s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += a[i];
      sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else if (KIND == 3) {
      uint32_t a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x + i; b[i] = i; }
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint64_t p = static_cast<uint64_t>(a[i]) * 0xD2511F53u;
          a[i] = static_cast<uint32_t>(p >> 32) ^ b[i];
          b[i] = static_cast<uint32_t>(p);
        }
      uint32_t s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += a[i] + b[i];
      sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else if (KIND == 4) {
      int a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __dp4a(a[i], 0x01020304, a[(i + 3) & 7]);
      int s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += a[i];
      sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else if (KIND == 5 || (KIND == 6 && (warp & 1))) {
      // DMMA m8n8k4 chains (4 independent accumulators)
      double acc[4][2];
#pragma unroll
      for (int i = 0; i < 4; ++i) { acc[i][0] = 0.0; acc[i][1] = 0.0; }
      const double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
      for (int it = 0; it < iters / 4; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
      double s = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
      sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    } else {
      uint32_t a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7 + i;
      for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t d;
          asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(a[i]), "r"(a[(i + 1) & 7]));
          a[i] = d ^ (a[i] + 0x9E3779B9u);
        }
      uint32_t s = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += a[i];
      sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    }
    long long t1 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = t1 - t0;   // warp 1 (DMMA in KIND 6)
    if (threadIdx.x == 64 && blockIdx.x == 0) out[1] = t1 - t0;   // warp 2 (ALU in KIND 6)
  }
  if (threadIdx.x == 0 && MODE == 1)
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}
template <int MODE, int KIND>
long long run(long long* out, double* sink, int tiles, int iters) {
  cudaFuncSetAttribute(k<MODE, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k<MODE, KIND><<<148, 288, 32768>>>(tiles, iters, out, sink);
  cudaDeviceSynchronize();
  return out[0];
}
int main() {
  long long* out; double* sink;
  cudaMallocManaged(&out, 64);
  cudaMalloc(&sink, 148 * 288 * 8);
  const int tiles = 4000, iters = 4000;
  printf("side warps: 8 x (8 chains x %d iters)\n", iters);
  printf("DFMA alone        %lld cycles\n", run<0, 0>(out, sink, tiles, iters));
  printf("DFMA + int8 MMA   %lld cycles\n", run<1, 0>(out, sink, tiles, iters));
  printf("ALU alone         %lld cycles\n", run<0, 1>(out, sink, tiles, iters));
  printf("ALU + int8 MMA    %lld cycles\n", run<1, 1>(out, sink, tiles, iters));
  printf("FFMA alone        %lld cycles\n", run<0, 2>(out, sink, tiles, iters));
  printf("FFMA + int8 MMA   %lld cycles\n", run<1, 2>(out, sink, tiles, iters));
  printf("IMAD.WIDE alone   %lld cycles\n", run<0, 3>(out, sink, tiles, iters));
  printf("IMAD.WIDE + MMA   %lld cycles\n", run<1, 3>(out, sink, tiles, iters));
  printf("IDP4A alone       %lld cycles\n", run<0, 4>(out, sink, tiles, iters));
  printf("IDP4A + MMA       %lld cycles\n", run<1, 4>(out, sink, tiles, iters));
  printf("DMMA alone        %lld cycles\n", run<0, 5>(out, sink, tiles, iters));
  printf("DMMA + int8 MMA   %lld cycles\n", run<1, 5>(out, sink, tiles, iters));
  long long d0 = run<0, 6>(out, sink, tiles, iters); long long a0 = out[1];
  printf("DMMA|ALU mix      DMMA warps %lld, ALU warps %lld cycles\n", d0, a0);
  long long d1 = run<1, 6>(out, sink, tiles, iters); long long a1 = out[1];
  printf("DMMA|ALU + MMA    DMMA warps %lld, ALU warps %lld cycles\n", d1, a1);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
