// Stream memory operations (driver API, resolved through the runtime's
// driver entry points so the library keeps linking against cudart only):
// a copy stream publishes per-block "resident" flags that a running
// persistent kernel polls, and waits on the kernel's per-block completion
// counters before copying finished blocks back -- host<->device traffic
// overlapped with the factorization / selected inversion instead of
// serialised around them.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace stbta {

struct MemOps {
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  bool ok = false;
};

// Resolved once per process; ok == false when the driver lacks them.
const MemOps& memops();

// cuTensorMapEncodeTiled (driver), nullptr when unavailable.
using TensorMapEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                       const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                       const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                       CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
TensorMapEncodeFn tensor_map_encode();

inline int memops_write(cudaStream_t st, const void* addr, unsigned v) {
  const MemOps& m = memops();
  if (!m.ok) return (int)cudaErrorNotSupported;
  return (int)m.write32((CUstream)st, (CUdeviceptr)addr, v, 0 /* CU_STREAM_WRITE_VALUE_DEFAULT */);
}
// wait until (int)(*addr - v) >= 0
inline int memops_wait_geq(cudaStream_t st, const void* addr, unsigned v) {
  const MemOps& m = memops();
  if (!m.ok) return (int)cudaErrorNotSupported;
  return (int)m.wait32((CUstream)st, (CUdeviceptr)addr, v, 0 /* CU_STREAM_WAIT_VALUE_GEQ */);
}

}  // namespace stbta
