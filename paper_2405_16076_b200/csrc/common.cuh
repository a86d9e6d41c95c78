// Shared device helpers of liboid (product side).  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace oid {

constexpr int kThreads = 256;

// Philox4x32-10 (reading R1).  One call = 4 x 32-bit words.
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#ifdef __CUDA_ARCH__
  const uint64_t p = static_cast<uint64_t>(a) * b;   // one IMAD.WIDE.U32
  lo = static_cast<uint32_t>(p);
  hi = static_cast<uint32_t>(p >> 32);
#else
  uint64_t p = static_cast<uint64_t>(a) * b;
  lo = static_cast<uint32_t>(p);
  hi = static_cast<uint32_t>(p >> 32);
#endif
}

__host__ __device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c0, hi0, lo0);
    mulhilo32(0xCD9E8D57u, c2, hi1, lo1);
    const uint32_t n0 = hi1 ^ c1 ^ k0;
    const uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

// Selection draw u(e, i, x) = (w0 >> 8) * 2^-24 at counter (e, i, x, tag = 1) (reading R6).
__device__ __forceinline__ double select_uniform(uint32_t epoch, uint32_t slot, uint32_t x, uint32_t k0, uint32_t k1) {
  U4 w = philox4x32_10(epoch, slot, x, 1u, k0, k1);
  return static_cast<double>(w.x >> 8) * 0x1p-24;
}

// Deterministic block-wide sum of one double (fixed tree order). All threads get the result.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red /* NT/32 doubles */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = red[0];
#pragma unroll
  for (int i = 1; i < NT / 32; ++i) s = fmax(s, red[i]);
  return s;
}

}  // namespace oid
