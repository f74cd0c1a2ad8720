// Probe: register layout of ldmatrix.m16n16.x1.trans.b8 (sm_100a LDSM.8.MT1616).
// smem byte (r, c) of a 16x16 matrix (row stride 16 B) holds (r << 4) | c.
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* o) {
  __shared__ __align__(128) uint8_t sm[256];
  for (int i = threadIdx.x; i < 256; i += 32) sm[i] = (uint8_t)i;
  __syncwarp();
  uint32_t a = (uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x % 16) * 16;
  uint32_t r0, r1, n0, n1;
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(a));
  n0 = n1 = 0;
  o[threadIdx.x * 4] = r0; o[threadIdx.x * 4 + 1] = r1; o[threadIdx.x * 4 + 2] = n0; o[threadIdx.x * 4 + 3] = n1;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 512);
  k<<<1, 32>>>(d);
  uint32_t h[128]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  for (int t = 0; t < 32; ++t) {
    printf("lane %2d trans:", t);
    for (int w = 0; w < 2; ++w) for (int b = 0; b < 4; ++b) { int v = (h[t * 4 + w] >> (8 * b)) & 255; printf(" (%2d,%2d)", v >> 4, v & 15); }
    printf("   plain:");
    for (int w = 2; w < 4; ++w) for (int b = 0; b < 4; ++b) { int v = (h[t * 4 + w] >> (8 * b)) & 255; printf(" (%2d,%2d)", v >> 4, v & 15); }
    printf("\n");
  }
}
