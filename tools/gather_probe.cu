// Probe: achievable HBM bandwidth for gathering rows of 128 B / 256 B (one KV head
// of one cache slot) in a random row order, with no math, three ways:
//   tma   - per-warp ring of gather4 TMA copies into smem (mbarrier completion)
//   ldgsts- per-warp ring of cp.async 16 B copies (wait_group pipelining)
//   ldg   - plain 16 B loads into registers, 4 rows in flight per lane group
// Grid: one CTA of 4 warps per 512 gathered rows, as in k2_attend_mma.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

constexpr int kRowsPerCta = 512;
constexpr int kWarps = 4;
constexpr int kTile = 16;
constexpr int kStages = 3;

__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(n)); }
__device__ __forceinline__ void mbar_tx(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t p) {
  asm volatile("{\n.reg .pred q;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W%=;\n}" ::"r"(b), "r"(p) : "memory");
}
__device__ __forceinline__ void g4(uint32_t dst, const CUtensorMap* m, int4 r, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
               ::"r"(dst), "l"((uint64_t)m), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(bar) : "memory");
}

template <int ROWB>
__global__ void __launch_bounds__(128) k_tma(const __grid_constant__ CUtensorMap m, const int* __restrict__ perm, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[kWarps * kStages];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int* rows = perm + (size_t)blockIdx.x * kRowsPerCta;
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(sm) + warp * kStages * kTile * ROWB;
  const uint32_t bb = (uint32_t)__cvta_generic_to_shared(bars) + warp * kStages * 8;
  if (lane == 0) { for (int s = 0; s < kStages; ++s) mbar_init(bb + 8 * s, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  const int ntiles = kRowsPerCta / kTile;
  auto issue = [&](int k, int s) {
    mbar_tx(bb + 8 * s, kTile * ROWB);
    for (int g = 0; g < kTile; g += 4) g4(ring + s * kTile * ROWB + g * ROWB, &m, *reinterpret_cast<const int4*>(rows + k * kTile + g), bb + 8 * s);
  };
  if (lane == 0) for (int i = 0; i < kStages; ++i) issue(warp + kWarps * i, i);
  int acc = 0;
  for (int it = 0; warp + kWarps * it < ntiles; ++it) {
    const int s = it % kStages;
    mbar_wait(bb + 8 * s, (it / kStages) & 1);
    acc += *reinterpret_cast<const int*>(sm + (warp * kStages + s) * kTile * ROWB + lane * 4);
    __syncwarp();
    const int kn = warp + kWarps * (it + kStages);
    if (lane == 0 && kn < ntiles) { asm volatile("fence.proxy.async.shared::cta;"); issue(kn, s); }
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int ROWB>
__global__ void __launch_bounds__(128) k_ldgsts(const uint8_t* __restrict__ base, const int* __restrict__ perm, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int* rows = perm + (size_t)blockIdx.x * kRowsPerCta;
  uint8_t* ring = sm + warp * kStages * kTile * ROWB;
  constexpr int CPR = ROWB / 16;                 // 16 B chunks per row
  constexpr int RPI = 32 / CPR;                  // rows per warp instruction
  const int ntiles = kRowsPerCta / kTile;
  auto issue = [&](int k, int s) {
    for (int r = lane / CPR; r < kTile; r += RPI) {
      const uint8_t* src = base + (size_t)rows[k * kTile + r] * ROWB + (lane % CPR) * 16;
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + s * kTile * ROWB + r * ROWB + (lane % CPR) * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int i = 0; i < kStages; ++i) if (warp + kWarps * i < ntiles) issue(warp + kWarps * i, i); else asm volatile("cp.async.commit_group;");
  int acc = 0;
  for (int it = 0; warp + kWarps * it < ntiles; ++it) {
    const int s = it % kStages;
    asm volatile("cp.async.wait_group %0;" ::"n"(kStages - 1) : "memory");
    __syncwarp();
    acc += *reinterpret_cast<const int*>(ring + s * kTile * ROWB + lane * 4);
    __syncwarp();
    const int kn = warp + kWarps * (it + kStages);
    if (kn < ntiles) issue(kn, s); else asm volatile("cp.async.commit_group;");
  }
  if (acc == 0x12345678) sink[0] = acc;
}

template <int ROWB>
__global__ void __launch_bounds__(128) k_ldg(const uint8_t* __restrict__ base, const int* __restrict__ perm, int* sink) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int* rows = perm + (size_t)blockIdx.x * kRowsPerCta;
  constexpr int CPR = ROWB / 16, RPI = 32 / CPR, U = 8;
  uint32_t acc = 0;
  for (int r0 = warp * RPI * U; r0 < kRowsPerCta; r0 += kWarps * RPI * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * RPI + lane / CPR;
      v[u] = __ldg(reinterpret_cast<const uint4*>(base + (size_t)rows[r] * ROWB) + lane % CPR);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678) sink[0] = acc;
}

int main() {
  const size_t total = 2048ull << 20;   // 2 GiB of rows
  uint8_t* buf; cudaMalloc(&buf, total); cudaMemset(buf, 1, total);
  int* sink; cudaMalloc(&sink, 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rowb : {128, 256}) {
    const int nrows = (int)(total / rowb);
    std::vector<int> perm(nrows);
    for (int i = 0; i < nrows; ++i) perm[i] = i;
    for (int mode = 0; mode < 2; ++mode) {
      if (mode == 1) { std::mt19937 g(1); std::shuffle(perm.begin(), perm.end(), g); }
      int* dperm; cudaMalloc(&dperm, (size_t)nrows * 4);
      cudaMemcpy(dperm, perm.data(), (size_t)nrows * 4, cudaMemcpyHostToDevice);
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)rowb, (cuuint64_t)nrows}, str[1] = {(cuuint64_t)rowb};
      cuuint32_t box[2] = {(cuuint32_t)rowb, 1}, es[2] = {1, 1};
      ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, str, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int grid = nrows / kRowsPerCta;
      const int smem = kWarps * kStages * kTile * rowb;
      for (int kind = 0; kind < 3; ++kind) {
        auto launch = [&]() {
          if (kind == 0) { if (rowb == 128) k_tma<128><<<grid, 128, smem>>>(m, dperm, sink); else k_tma<256><<<grid, 128, smem>>>(m, dperm, sink); }
          if (kind == 1) { if (rowb == 128) k_ldgsts<128><<<grid, 128, smem>>>(buf, dperm, sink); else k_ldgsts<256><<<grid, 128, smem>>>(buf, dperm, sink); }
          if (kind == 2) { if (rowb == 128) k_ldg<128><<<grid, 128>>>(buf, dperm, sink); else k_ldg<256><<<grid, 128>>>(buf, dperm, sink); }
        };
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 5.0 * ((double)nrows * rowb + (double)nrows * 4);
        printf("row %3d B  %-8s %-6s  %7.1f GB/s  (%s)\n", rowb, mode ? "random" : "linear",
               kind == 0 ? "tma" : kind == 1 ? "ldgsts" : "ldg", bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
      cudaFree(dperm);
    }
  }
  return 0;
}
