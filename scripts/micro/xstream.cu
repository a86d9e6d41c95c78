// Streaming read of a column-major m x 32 fp64 block (C3 K1 shape) into shared memory, by method:
//   0: TMA 2-D boxes {16 rows, 32 cols}, 128B swizzle (K1F / K1 exact)
//   1: TMA 2-D boxes {64 rows, 32 cols}, no swizzle (512-byte lines)
//   2: TMA 2-D boxes {64 rows, 8 cols}, no swizzle, 4 per tile
//   3: LDG.128 by 16 warps (each warp one column run of 512 B), register-only consumer
// One persistent CTA per SM, tiles of 64 rows dealt round-robin, NST stages of 16 KB.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_2405_16076_b200/csrc/sm100.cuh"
using namespace oid::k1tc;

constexpr int NST = 8;
struct Sh { uint64_t full[NST], empty[NST]; };

template <int MODE>
__global__ void __launch_bounds__(512, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const double* X, int64_t m, int64_t ld,
                                                        double* out) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ Sh sh;
  uint8_t* buf = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles = (m + 63) / 64;
  const int nt = static_cast<int>((tiles - blockIdx.x + gridDim.x - 1) / gridDim.x);
  double acc = 0.0;
  if (MODE == 3) {
    // warps 0..15: warp w reads columns 2w, 2w+1 of each tile (512 B each, 8 tiles in flight)
    for (int t = 0; t < nt; t += 4) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t row = (blockIdx.x + int64_t(t + u) * gridDim.x) * 64 + 2 * lane;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int col = 2 * warp + cc;
          v[2 * u + cc] = (t + u < nt && row < m) ? __ldg(reinterpret_cast<const double2*>(X + col * ld + row)) : make_double2(0, 0);
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y;
    }
    if (acc == 1.2345) out[0] = acc;
    return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&sh.full[s], 1); mbar_init(&sh.empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    for (int t = 0; t < nt; ++t) {
      const int s = t % NST;
      if (t >= NST) mbar_wait(&sh.empty[s], ((t / NST) - 1) & 1);
      mbar_arrive_expect_tx_e(&sh.full[s], 16384);
      const int row0 = static_cast<int>((blockIdx.x + int64_t(t) * gridDim.x) * 64);
      uint8_t* dst = buf + s * 16384;
      if (MODE == 0) {
        for (int bx = 0; bx < 4; ++bx) tma_load_2d_e(dst + bx * 4096, &map, &sh.full[s], row0 + 16 * bx, 0);
      } else if (MODE == 1) {
        tma_load_2d_e(dst, &map, &sh.full[s], row0, 0);
      } else {
        for (int bx = 0; bx < 4; ++bx) tma_load_2d_e(dst + bx * 4096, &map, &sh.full[s], row0, 8 * bx);
      }
    }
  } else if (warp >= 8) {
    for (int t = 0; t < nt; ++t) {
      const int s = t % NST;
      mbar_wait(&sh.full[s], (t / NST) & 1);
      const double2 v = *reinterpret_cast<const double2*>(buf + s * 16384 + (warp - 8) * 2048 + lane * 64);
      acc += v.x;
      __syncwarp();
      if (lane == 0) mbar_arrive(&sh.empty[s]);
    }
    if (acc == 1.2345) out[0] = acc;
  }
}

typedef CUresult (*PFN)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int64_t m = 14266368, ncol = 32;
  double* X;
  cudaMalloc(&X, m * ncol * 8);
  cudaMemset(X, 0, m * ncol * 8);
  double* out;
  cudaMalloc(&out, 8);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  PFN enc = reinterpret_cast<PFN>(p);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 4; ++mode) {
    for (int prom = 0; prom < 3; ++prom) {
      if (mode == 3 && prom > 0) continue;
      CUtensorMap map;
      const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)ncol};
      const cuuint64_t strides[1] = {(cuuint64_t)m * 8};
      cuuint32_t box[2] = {16, 32};
      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
      if (mode == 1) { box[0] = 64; sw = CU_TENSOR_MAP_SWIZZLE_NONE; }
      if (mode == 2) { box[0] = 64; box[1] = 8; sw = CU_TENSOR_MAP_SWIZZLE_NONE; }
      const cuuint32_t es[2] = {1, 1};
      CUtensorMapL2promotion pr = prom == 0 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : (prom == 1 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("mode %d encode failed %d\n", mode, (int)r); continue; }
      auto fn = mode == 0 ? stream_kernel<0> : mode == 1 ? stream_kernel<1> : mode == 2 ? stream_kernel<2> : stream_kernel<3>;
      const int smem = NST * 16384 + 1024;
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      float best = 1e9;
      for (int it = 0; it < 5; ++it) {
        cudaEventRecord(e0);
        fn<<<sms, 512, smem>>>(map, X, m, m, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("mode %d prom %d: %.3f ms  %.0f GB/s  (%s)\n", mode, prom, best, m * ncol * 8 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
