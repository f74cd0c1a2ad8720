// Decode-loop glue: the fused QKV projection's bf16 output row
// [q | k | v] per sequence is split and converted to the engine's fp16 inputs in
// one pass (q for K2, k/v for the step's append), instead of three strided copies.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "ckv_internal.cuh"

namespace {

// one thread = 8 consecutive elements (16 B bf16 in, 16 B fp16 out); grid-stride over B rows
__global__ void k_qkv_split(const __nv_bfloat16* __restrict__ qkv, int B, int d, int kvd,
                            __half* __restrict__ q, __half* __restrict__ k, __half* __restrict__ v) {
  const int w = d + 2 * kvd;
  const int per_row = w / 8;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < B * per_row; idx += gridDim.x * blockDim.x) {
    const int b = idx / per_row, c = (idx - b * per_row) * 8;
    const uint4 in = *reinterpret_cast<const uint4*>(qkv + (size_t)b * w + c);
    const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&in);
    uint4 o;
    __half2* o2 = reinterpret_cast<__half2*>(&o);
#pragma unroll
    for (int j = 0; j < 4; ++j) o2[j] = __float22half2_rn(__bfloat1622float2(h2[j]));
    __half* dst = c < d ? q + (size_t)b * d + c
                : c < d + kvd ? k + (size_t)b * kvd + (c - d) : v + (size_t)b * kvd + (c - d - kvd);
    *reinterpret_cast<uint4*>(dst) = o;
  }
}

}  // namespace

extern "C" int ckv_qkv_split(const void* qkv, int32_t batch, int32_t d, int32_t kvd, void* q, void* k, void* v,
                             void* stream) {
  if (!qkv || !q || !k || !v || batch <= 0 || d <= 0 || kvd <= 0) return CKV_EINVAL;
  if ((d | kvd) % 8 || ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(q) |
                         reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) % 16))
    return CKV_EINVAL;
  const int total = batch * ((d + 2 * kvd) / 8);
  const int threads = 256, blocks = (total + threads - 1) / threads;
  k_qkv_split<<<blocks, threads, 0, (cudaStream_t)stream>>>(reinterpret_cast<const __nv_bfloat16*>(qkv), batch, d,
                                                            kvd, (__half*)q, (__half*)k, (__half*)v);
  return cudaGetLastError() == cudaSuccess ? CKV_OK : CKV_ECUDA;
}
