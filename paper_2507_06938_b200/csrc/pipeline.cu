// Pipelined host <-> device transfers of BTA matrices (C ABI).
//
// The reference keeps every matrix in host memory (numpy); its drop-in here
// is a BTAMatrix built from a host buffer, factorized, solved and selected-
// inverted, with the inverse read back to the host (bta.py:50-359).  Instead
// of copying 3.2 GB up front and back at the end, the upload is split into
// time-block chunks on a copy stream, each followed by a flag write that the
// POBTAF task graph polls before it touches that block (stbta_pobtaf_ready),
// and the inverse streams back block by block as the POBTASI recursion
// finishes them (stbta_pobtasi_stream_out, pobtasi.cu).
#include <cstdint>

#include "../../include/stbta.h"
#include "common.cuh"
#include "memops.cuh"

namespace stbta {

const MemOps& memops() {
  static MemOps m = [] {
    MemOps r;
    void* w = nullptr;
    void* q = nullptr;
    cudaDriverEntryPointQueryResult s1 = cudaDriverEntryPointSymbolNotFound, s2 = s1;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &s1) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &q, cudaEnableDefault, &s2) == cudaSuccess &&
        s1 == cudaDriverEntryPointSuccess && s2 == cudaDriverEntryPointSuccess && w && q) {
      r.write32 = reinterpret_cast<CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int)>(w);
      r.wait32 = reinterpret_cast<CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int)>(q);
      r.ok = true;
    }
    cudaGetLastError();
    return r;
  }();
  return m;
}

TensorMapEncodeFn tensor_map_encode() {
  static TensorMapEncodeFn f = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult st = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &st) != cudaSuccess ||
        st != cudaDriverEntryPointSuccess)
      fn = nullptr;
    cudaGetLastError();
    return reinterpret_cast<TensorMapEncodeFn>(fn);
  }();
  return f;
}

}  // namespace stbta

using namespace stbta;

extern "C" {

int stbta_stream_memops_supported(void) { return memops().ok ? 1 : 0; }

int stbta_upload_blocks(double* dst, const double* src_host, int n, int b, int a, unsigned* ready,
                        unsigned epoch, void* stream) {
  if (dst == nullptr || src_host == nullptr || ready == nullptr || n < 1 || b < 1 || a < 0)
    return STBTA_EARG;
  if (!memops().ok) return (int)cudaErrorNotSupported;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long long bb = (long long)b * b;
  const long long o_low = (long long)n * bb, o_arr = o_low + (long long)(n - 1) * bb;
  const long long o_tip = o_arr + (long long)n * a * b;
  int e;
  if (a > 0 && (e = (int)cudaMemcpyAsync(dst + o_tip, src_host + o_tip, (size_t)a * a * sizeof(double),
                                         cudaMemcpyHostToDevice, st)))
    return e;  // the tip travels with chunk 0: every block's arrow update touches it
  for (int t = 0; t < n; ++t) {
    if ((e = (int)cudaMemcpyAsync(dst + t * bb, src_host + t * bb, bb * sizeof(double),
                                  cudaMemcpyHostToDevice, st)))
      return e;
    if (t < n - 1 && (e = (int)cudaMemcpyAsync(dst + o_low + t * bb, src_host + o_low + t * bb,
                                               bb * sizeof(double), cudaMemcpyHostToDevice, st)))
      return e;
    if (a > 0) {
      const long long ab = (long long)a * b;
      if ((e = (int)cudaMemcpyAsync(dst + o_arr + t * ab, src_host + o_arr + t * ab,
                                    ab * sizeof(double), cudaMemcpyHostToDevice, st)))
        return e;
    }
    if ((e = memops_write(st, ready + t, epoch))) return e;
  }
  return 0;
}

}  // extern "C"
