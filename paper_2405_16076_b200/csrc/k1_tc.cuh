// K1, tensor-core variant (tcgen05 kind::i8) — interface.  Implementation in progress; until
// it lands k1tc_supported() returns false and OID_K1_AUTO selects the CUDA-core kernel.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace oid {

struct K1TcArgs {
  const void* X;
  int64_t ld;
  int ncols;
  int64_t row_begin, row_end;
  int ell;
  uint32_t key0, key1;
  double scale;
  bool f64;
  char* ws;
  double* out;
  unsigned* flags;
  int num_sms;
};

inline size_t k1tc_workspace_bytes(int /*ell*/, int /*b_max*/, int64_t /*m_loc*/, bool /*f64*/) { return 256; }
inline bool k1tc_supported(int /*ell*/, int /*b_max*/, bool /*f64*/) { return false; }
inline cudaError_t k1tc_init_tables(const int32_t* /*q*/, cudaStream_t /*st*/) { return cudaSuccess; }
inline cudaError_t k1tc_launch(const K1TcArgs& /*a*/, cudaStream_t /*st*/, int* nlaunch) {
  *nlaunch = 0;
  return cudaErrorNotSupported;
}

}  // namespace oid
