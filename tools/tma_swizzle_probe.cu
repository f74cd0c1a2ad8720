// Probe: how does tile::gather4 + SWIZZLE_128B place 4 gathered 128-byte rows in
// shared memory, for destinations at 1024-aligned and 512-offset addresses?
// Prints, for each smem 16-byte chunk, which (row, chunk) of global it holds.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>

__global__ void probe(const __grid_constant__ CUtensorMap map, uint32_t* out, int off_bytes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 4096 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0xffffffffu;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512));
    uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + off_bytes);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(dst), "l"((uint64_t)&map), "r"(0), "r"(5), "r"(9), "r"(2), "r"(7), "r"(b) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048 / 4; i += blockDim.x) out[i] = reinterpret_cast<uint32_t*>(sm)[i];
}

int main() {
  const int rows = 16, cols = 128;  // uint8 rows of 128 bytes
  uint8_t h[rows * cols];
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint8_t)(r * 16 + c / 16);  // tag = row*16 + chunk
  void* g; cudaMalloc(&g, sizeof(h)); cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  uint32_t* out; cudaMalloc(&out, 2048);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows}, strides[1] = {cols};
  cuuint32_t box[2] = {cols, 1}, es[2] = {1, 1};
  CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, g, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int off : {0, 512, 128}) {
    cudaMemset(out, 0, 2048);
    probe<<<1, 128, 4096>>>(m, out, off);
    cudaError_t e = cudaDeviceSynchronize();
    uint8_t res[2048]; cudaMemcpy(res, out, 2048, cudaMemcpyDeviceToHost);
    printf("dst offset %d: %s\n", off, cudaGetErrorString(e));
    for (int line = 0; line < 12; ++line) {
      printf("  line %2d:", line);
      for (int ch = 0; ch < 8; ++ch) { uint8_t t = res[line * 128 + ch * 16]; if (t == 0xff) printf("  --"); else printf(" %d.%d", t / 16, t % 16); }
      printf("\n");
    }
    if (e != cudaSuccess) return 0;
  }
  return 0;
}
