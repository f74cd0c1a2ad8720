// Probe: tcgen05.mma kind::i8 with the four operand layouts the INT8 attention path uses.
//   S[t][n] = sum_k K[t][k] * Q[n][k]   A = K  (SW128 K-major),  B = Q (plain K-major)
//   O[m][n] = sum_t V[t][m] * P[t][n]   A = V^T (SW128 MN-major), B = P (plain MN-major, u8)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_i8_probe tools/tc_i8_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_2605_24786_b200/csrc/tc_i8.cuh"
using namespace ckv;

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(bar),
      "r"(parity) : "memory");
}

template <int N>
__global__ void probe(const int8_t* K, const int8_t* Q, const int8_t* V, const uint8_t* P, int* S, int* O) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sK = sm;                 // 16 KB SW128
  uint8_t* sV = sm + 16384;         // 16 KB SW128
  uint8_t* sQ = sm + 32768;         // N x 128 plain K-major
  uint8_t* sP = sm + 40960;         // 128 x N plain MN-major
  uint32_t* tslot = (uint32_t*)(sm + 49152);
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(sm + 49152 + 16);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int i = t; i < 128 * 128; i += 128) {
    const int r = i / 128, b = i % 128;
    const int off = r * 128 + ((((b >> 4) ^ (r & 7))) << 4) + (b & 15);
    sK[off] = (uint8_t)K[i];
    sV[off] = (uint8_t)V[i];
  }
  for (int i = t; i < N * 128; i += 128) {
    const int n = i / 128, k = i % 128;
    sQ[(n / 8) * 1024 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = (uint8_t)Q[i];
  }
  for (int i = t; i < 128 * N; i += 128) {
    const int k = i / N, n = i % N;
    sP[(n / 16) * 2048 + (k / 8) * 128 + (k % 8) * 16 + (n % 16)] = P[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tc::alloc((uint32_t)__cvta_generic_to_shared(tslot), 64);
  if (t == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = *tslot;
  const uint32_t aK = (uint32_t)__cvta_generic_to_shared(sK), aV = (uint32_t)__cvta_generic_to_shared(sV);
  const uint32_t aQ = (uint32_t)__cvta_generic_to_shared(sQ), aP = (uint32_t)__cvta_generic_to_shared(sP);
  if (t == 0) {
    constexpr uint32_t iqk = tc::idesc_i8(128, N, true, true, false, false);
    constexpr uint32_t ipv = tc::idesc_i8(128, N, true, false, true, true);
    for (int ks = 0; ks < 4; ++ks)
      tc::mma_i8(tm, tc::sdesc(aK + 32 * ks, 16, 1024, tc::kSW128), tc::sdesc(aQ + 256 * ks, 128, 1024, tc::kInterleave),
                 iqk, ks > 0);
    for (int ks = 0; ks < 4; ++ks)
      tc::mma_i8(tm + 32, tc::sdesc(aV + 4096 * ks, 8192, 1024, tc::kSW128),
                 tc::sdesc(aP + 512 * ks, 128, 2048, tc::kInterleave), ipv, ks > 0);
    tc::commit(bar);
  }
  __syncwarp();
  mbar_wait(bar, 0);
  tc::fence_after();
  for (int h = 0; h < N / 16; ++h) {
    int r[16];
    tc::ld16(tm + ((uint32_t)(32 * warp) << 16) + 16 * h, r);
    tc::wait_ld();
    for (int j = 0; j < 16; ++j) S[(32 * warp + lane) * N + 16 * h + j] = r[j];
    tc::ld16(tm + ((uint32_t)(32 * warp) << 16) + 32 + 16 * h, r);
    tc::wait_ld();
    for (int j = 0; j < 16; ++j) O[(32 * warp + lane) * N + 16 * h + j] = r[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) { tc::fence_after(); tc::dealloc(tm, 64); }
}

template <int N>
int run() {
  int8_t *K, *Q, *V; uint8_t* P; int *S, *O;
  cudaMallocManaged(&K, 16384); cudaMallocManaged(&V, 16384); cudaMallocManaged(&Q, N * 128);
  cudaMallocManaged(&P, 128 * N); cudaMallocManaged(&S, 128 * N * 4); cudaMallocManaged(&O, 128 * N * 4);
  srand(N);
  for (int i = 0; i < 16384; ++i) { K[i] = (int8_t)(rand() % 255 - 127); V[i] = (int8_t)(rand() % 255 - 127); }
  for (int i = 0; i < N * 128; ++i) Q[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < N * 128; ++i) P[i] = (uint8_t)(rand() % 256);
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50000);
  probe<N><<<1, 128, 50000>>>(K, Q, V, P, S, O);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d cuda error %s\n", N, cudaGetErrorString(e)); return 1; }
  int bad = 0;
  for (int t = 0; t < 128; ++t)
    for (int n = 0; n < N; ++n) {
      long s = 0, o = 0;
      for (int k = 0; k < 128; ++k) s += (long)K[t * 128 + k] * Q[n * 128 + k];
      for (int k = 0; k < 128; ++k) o += (long)V[k * 128 + t] * P[k * N + n];
      if (s != S[t * N + n]) { if (bad < 5) printf("S[%d][%d] %ld vs %d\n", t, n, s, S[t * N + n]); ++bad; }
      if (o != O[t * N + n]) { if (bad < 5) printf("O[%d][%d] %ld vs %d\n", t, n, o, O[t * N + n]); ++bad; }
    }
  printf("N=%d mismatches %d\n", N, bad);
  return bad != 0;
}

int main() { return run<16>() | run<32>(); }
