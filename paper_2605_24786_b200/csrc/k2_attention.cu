// K2 — split-K online-softmax decode attention over the mixed FP16/INT8 cache,
// plus the combine / head-mean epilogue that stages the EMA input.
//
// Replaces tiled_attention (attention.py:60-102), LayerCache.read_block +
// dequantize (cache.py:238-252, quantizer.py:37-39) and the head-mean of
// update_attention_ema (cache.py:171). Grid = (split, kv head, cache): each CTA
// streams kSplitTokens entries of one KV head and serves all G = Hq/Hkv query
// heads of the group from the same K/V bytes (GQA), so every K/V byte is read
// from HBM exactly once per step.
//
// Warp-specialised TMA pipeline. One producer thread stages each group of 4
// gathered entries with a Blackwell `tile::gather4` TMA (4 arbitrary rows of
// the 2-D [slot*Hkv+head][D] tensor map per instruction, SASS UTMALDG) — the K
// and V rows of this KV head at the entries' physical slots, 2*D bytes (FP16)
// or D bytes (INT8 codes) each — completing on the stage's mbarrier
// (arrive.expect_tx). 1-D `cp.async.bulk` (UBLKCP) covers the one group per
// cache that straddles the INT8/FP16 boundary. A
// kStages-deep ring keeps up to kStages*STAGE_TOK*4*D bytes in flight per CTA
// independent of register pressure. Warps 0-3 consume: a token row is spread
// over LPR = D/8 lanes holding 8 dims; q.k partials for the U*G (token, head)
// pairs are reduced with a recursive-halving butterfly, the running max /
// rescale uses a warp-private smem tile, P.V accumulates with packed fp32x2
// FMA (FFMA2, sm_100). INT8 codes are widened exactly (PRMT + FADD) and
// dequantised code*scale in fp32 as the reference does; the segment's fp32
// scale row is cached in registers while consecutive entries share a segment.
// Entry slot and segment ids are staged into smem once per CTA, so no load
// waits on another load.
//
// Split partials (m, z, acc) go to scratch; k2_combine merges them (out) and
// turns the raw fp32 scores into the normalised weights the EMA consumes,
// summing heads sequentially in fp64 and dividing by Hq (cache.py:171's
// NumPy axis-0 mean) into abar[c][i].
#include <algorithm>
#include <cstdlib>
#include "ckv_internal.cuh"
#include <cstdio>
#include "tc_i8.cuh"

namespace ckv {
namespace {

constexpr int kConsumerWarps = 4;
thread_local int g_k2_launches = 0;   // kernels the last launch_attend issued (ckv_launch_count)
constexpr int kStages = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

__host__ __device__ constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

template <int D, int G>
struct Tr {
  static constexpr int LPR = D / 8;                      // lanes per token row
  static constexpr int RPW = 32 / LPR;                   // rows per warp instruction
  static constexpr int U = D == 128 ? 4 : (D == 64 ? 2 : 1);
  static constexpr int TT = RPW * U;                     // tokens per consumer warp per stage
  static constexpr int STAGE_TOK = TT * kConsumerWarps;  // tokens per stage
  static constexpr int ROWB = 2 * D;                     // smem bytes per row slot
  static constexpr int STAGE_BYTES = STAGE_TOK * ROWB * 2;
  static constexpr int K = U * G;                        // (token, head) dots per lane group
  static constexpr int KP = pow2ceil(K);
  static constexpr int HS = ilog2(cmin(KP, LPR));        // halving steps
  static constexpr int CNT = KP >= LPR ? KP / LPR : 1;   // values held per lane afterwards
  static constexpr int REP = KP >= LPR ? 1 : LPR / KP;   // lanes holding the same value
  // smem carve-up (bytes)
  static constexpr int OFF_BAR = kStages * STAGE_BYTES;                 // 2*kStages mbarriers
  static constexpr int OFF_SLOT = OFF_BAR + 2 * kStages * 8;
  static constexpr int OFF_SEG = OFF_SLOT + kSplitTokens * 4;
  static constexpr int OFF_S = OFF_SEG + kSplitTokens * 4;              // sS[warps][G][TT]
  static constexpr int OFF_P = OFF_S + kConsumerWarps * G * TT * 4;     // sP
  static constexpr int SMEM = OFF_P + kConsumerWarps * G * TT * 4;
  static_assert(kConsumerWarps * G * (D + 2) * 4 <= kStages * STAGE_BYTES, "epilogue alias");
  static_assert(STAGE_TOK % 32 == 0, "producer lanes map to rows");
};

// Entry range of partial slot `part` of split `split` (see Dev::npart).
__device__ __forceinline__ void part_range(const Dev& d, int split, int part, int n, int nq, int& b, int& e) {
  const int s0 = split * kSplitTokens;
  int s1 = min(n, s0 + kSplitTokens);
  if (d.absorb) {
    // A cache at budget N + 1 (N a multiple of 512) would otherwise end in a 1-entry split: its
    // own CTA, partial slot and merge. A remainder r <= kAbsorbTokens of FP16 entries (no codes
    // part grows past 512, no bulk-codes split turns mixed) is read by the last full split.
    const int ns = n / kSplitTokens, r = n - ns * kSplitTokens;
    const int lim = d.cut_nq ? ns * kSplitTokens : (ns - 1) * kSplitTokens;
    if (ns >= 1 && r > 0 && r <= kAbsorbTokens && nq <= lim) {
      if (split == ns) { b = e = s0; return; }
      if (split == ns - 1) s1 = n;
    }
  }
  const int cut = d.cut_nq ? min(max(nq, s0), s1) : s1;
  b = part ? cut : s0;
  e = part ? s1 : cut;
}

union F2 {
  float2 f;
  unsigned long long u;
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  F2 x, y, z, r;
  x.f = a; y.f = b; z.f = c;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.u) : "l"(x.u), "l"(y.u), "l"(z.u));
  return r.f;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  F2 x, y, r;
  x.f = a; y.f = b;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(x.u), "l"(y.u));
  return r.f;
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  F2 x, y, r;
  x.f = a; y.f = b;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(x.u), "l"(y.u));
  return r.f;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar), "r"(parity) : "memory");
}
// Blackwell TMA row gather: 4 rows (arbitrary row coordinates) of a 2-D tensor
// map with a one-row box land back to back at dst.
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                            uint32_t bar, int col = 0) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

__device__ __forceinline__ void half8_to_f2(const uint4& w, float2 (&o)[4]) {
  o[0] = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
  o[1] = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
  o[2] = __half22float2(*reinterpret_cast<const __half2*>(&w.z));
  o[3] = __half22float2(*reinterpret_cast<const __half2*>(&w.w));
}

// 8 signed int8 codes -> 8 exact floats: bias to unsigned, splice into the
// mantissa of 2^23 (PRMT), subtract 2^23 + 128 (packed FADD2).
__device__ __forceinline__ void code8_to_f2(const uint2& w, float2 (&o)[4]) {
  const unsigned a = w.x ^ 0x80808080u, b = w.y ^ 0x80808080u;
  const float2 k = make_float2(-8388736.0f, -8388736.0f);
  o[0] = fadd2(make_float2(__int_as_float(__byte_perm(a, 0x4B000000u, 0x7440)),
                           __int_as_float(__byte_perm(a, 0x4B000000u, 0x7441))), k);
  o[1] = fadd2(make_float2(__int_as_float(__byte_perm(a, 0x4B000000u, 0x7442)),
                           __int_as_float(__byte_perm(a, 0x4B000000u, 0x7443))), k);
  o[2] = fadd2(make_float2(__int_as_float(__byte_perm(b, 0x4B000000u, 0x7440)),
                           __int_as_float(__byte_perm(b, 0x4B000000u, 0x7441))), k);
  o[3] = fadd2(make_float2(__int_as_float(__byte_perm(b, 0x4B000000u, 0x7442)),
                           __int_as_float(__byte_perm(b, 0x4B000000u, 0x7443))), k);
}

// fp32 scale rows (8 dims of K and of V) of the segment the lane's entry uses.
struct ScaleCache {
  int seg;
  float2 k[4], v[4];
};

__device__ __forceinline__ void load_scales(ScaleCache& sc, const Dev& d, int c, int h, int sg, int D, int rl) {
  if (sg == sc.seg) return;
  const size_t off = (((size_t)c * d.smax + sg) * d.Hkv + h) * D + rl * 8;
  const float4* kp = reinterpret_cast<const float4*>(d.ksc + off);
  const float4* vp = reinterpret_cast<const float4*>(d.vsc + off);
  const float4 k0 = __ldg(kp), k1 = __ldg(kp + 1), v0 = __ldg(vp), v1 = __ldg(vp + 1);
  sc.k[0] = make_float2(k0.x, k0.y); sc.k[1] = make_float2(k0.z, k0.w);
  sc.k[2] = make_float2(k1.x, k1.y); sc.k[3] = make_float2(k1.z, k1.w);
  sc.v[0] = make_float2(v0.x, v0.y); sc.v[1] = make_float2(v0.z, v0.w);
  sc.v[2] = make_float2(v1.x, v1.y); sc.v[3] = make_float2(v1.z, v1.w);
  sc.seg = sg;
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 3)
k2_attend_split(Dev d, const __grid_constant__ Maps maps, int c0, const __half* __restrict__ q, float qscale) {
  using T = Tr<D, G>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int c = c0 + blockIdx.z;
  const int h = blockIdx.y;
  const int split = blockIdx.x;
  const int n = d.len[c];
  const int begin = split * kSplitTokens;
  if (begin >= n) return;
  const int end = min(n, begin + kSplitTokens);
  const int ntok = end - begin;
  const int nst = (ntok + T::STAGE_TOK - 1) / T::STAGE_TOK;
  const int n8 = d.nq[c];   // INT8-codes prefix (single-entry segments are read from their FP16 rows)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t cbase = (size_t)c * d.cap;
  const uint32_t sbase = smem_u32(smem);
  int* s_slot = reinterpret_cast<int*>(smem + T::OFF_SLOT);
  int* s_seg = reinterpret_cast<int*>(smem + T::OFF_SEG);

  for (int j = threadIdx.x; j < ntok; j += kThreads) {
    s_slot[j] = __ldg(d.slot + cbase + begin + j);
    s_seg[j] = (begin + j < n8) ? __ldg(d.seg + cbase + begin + j) : -1;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(sbase + T::OFF_BAR + 8 * s, 1);                          // full: the producer thread
      mbar_init(sbase + T::OFF_BAR + 8 * (kStages + s), kConsumerWarps);  // empty
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ===== producer (one thread): gather4 TMA of the stage's K and V rows =====
    // Rows are grouped 4 at a time in smem blocks of 4*ROWB bytes: FP16 rows at
    // stride ROWB, INT8 rows at stride D (what gather4 writes). A group that
    // straddles the INT8/FP16 boundary or the end uses per-row 1-D bulk copies.
    if (lane == 0) {
      const size_t row = (size_t)d.Hkv * D;
      const int rbase = c * d.cap;   // row coordinate = (c*cap + slot)*Hkv + h
      for (int it = 0; it < nst; ++it) {
        const int s = it % kStages;
        const uint32_t full = sbase + T::OFF_BAR + 8 * s;
        if (it >= kStages) mbar_wait(sbase + T::OFF_BAR + 8 * (kStages + s), ((it / kStages) & 1) ^ 1);
        const int j = it * T::STAGE_TOK;
        const int t0 = begin + j;
        const int nrow = min(T::STAGE_TOK, end - t0);
        const int n8s = max(0, min(nrow, n8 - t0));   // INT8 rows of this stage: [0, n8s)
        mbar_arrive_tx(full, (uint32_t)(n8s * 2 * D + (nrow - n8s) * 4 * D));
        const uint32_t kb = sbase + s * T::STAGE_BYTES;
        const uint32_t vb = kb + T::STAGE_TOK * T::ROWB;
        for (int g0 = 0; g0 < nrow; g0 += 4) {
          const uint32_t ko = kb + g0 * T::ROWB, vo = vb + g0 * T::ROWB;
          const bool whole = g0 + 4 <= nrow;
          if (whole && (g0 + 4 <= n8s || g0 >= n8s)) {
            if (g0 >= n8s) {
              const int r0 = (rbase + s_slot[j + g0]) * d.Hkv + h, r1 = (rbase + s_slot[j + g0 + 1]) * d.Hkv + h;
              const int r2 = (rbase + s_slot[j + g0 + 2]) * d.Hkv + h, r3 = (rbase + s_slot[j + g0 + 3]) * d.Hkv + h;
              tma_gather4(ko, &maps.kf, r0, r1, r2, r3, full);
              tma_gather4(vo, &maps.vf, r0, r1, r2, r3, full);
            } else {   // code slots -> code rows
              const int r0 = code_row(rbase, s_slot[j + g0], d.Hkv, h), r1 = code_row(rbase, s_slot[j + g0 + 1], d.Hkv, h);
              const int r2 = code_row(rbase, s_slot[j + g0 + 2], d.Hkv, h), r3 = code_row(rbase, s_slot[j + g0 + 3], d.Hkv, h);
              tma_gather4(ko, &maps.kq, r0, r1, r2, r3, full);
              tma_gather4(vo, &maps.vq, r0, r1, r2, r3, full);
            }
          } else {
            for (int r = g0; r < min(g0 + 4, nrow); ++r) {
              const size_t off = ((size_t)rbase + s_slot[j + r]) * row + (size_t)h * D;
              if (r < n8s) {
                const size_t co = (size_t)code_row(rbase, s_slot[j + r], d.Hkv, h) * D;
                tma_row(ko + (r - g0) * D, d.kq + co, D, full);
                tma_row(vo + (r - g0) * D, d.vq + co, D, full);
              } else {
                tma_row(ko + (r - g0) * T::ROWB, d.kf + off, 2 * D, full);
                tma_row(vo + (r - g0) * T::ROWB, d.vf + off, 2 * D, full);
              }
            }
          }
        }
      }
    }
  } else {
    // ================= consumers =================
    const int rg = lane / T::LPR, rl = lane % T::LPR;
    const int Hq = d.Hq;
    float* sS = reinterpret_cast<float*>(smem + T::OFF_S) + warp * G * T::TT;
    float* sP = reinterpret_cast<float*>(smem + T::OFF_P) + warp * G * T::TT;

    float2 qv[G][4];
    {
      const __half* qp = q + ((size_t)(c - c0) * Hq + (size_t)h * G) * D + rl * 8;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        uint4 w = *reinterpret_cast<const uint4*>(qp + (size_t)g * D);
        half8_to_f2(w, qv[g]);
#pragma unroll
        for (int j = 0; j < 4; ++j) qv[g][j] = fmul2(qv[g][j], make_float2(qscale, qscale));
      }
    }
    float m[G], zp[G];
    float2 acc[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      m[g] = -INFINITY;
      zp[g] = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[g][j] = make_float2(0.f, 0.f);
    }
    ScaleCache sc;
    sc.seg = -1;
    float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.sld;

    for (int it = 0; it < nst; ++it) {
      const int s = it % kStages;
      mbar_wait(sbase + T::OFF_BAR + 8 * s, (it / kStages) & 1);
      const uint8_t* stK = smem + s * T::STAGE_BYTES;
      const uint8_t* stV = stK + T::STAGE_TOK * T::ROWB;
      const int tb = begin + it * T::STAGE_TOK + warp * T::TT;   // first token of this warp's slice
      const int rb = warp * T::TT;                               // its first row slot in the stage

      // ---- q.k partials -------------------------------------------------------------
      float v[T::KP];
#pragma unroll
      for (int k = 0; k < T::KP; ++k) v[k] = 0.f;
#pragma unroll
      for (int u = 0; u < T::U; ++u) {
        const int r = rb + u * T::RPW + rg;
        const int tok = tb + u * T::RPW + rg;
        float2 kx[4];
        if (tok < end) {
          if (tok < n8) {
            code8_to_f2(*reinterpret_cast<const uint2*>(stK + (r & ~3) * T::ROWB + (r & 3) * D + rl * 8), kx);
            load_scales(sc, d, c, h, s_seg[tok - begin], D, rl);
#pragma unroll
            for (int j = 0; j < 4; ++j) kx[j] = fmul2(kx[j], sc.k[j]);
          } else {
            half8_to_f2(*reinterpret_cast<const uint4*>(stK + r * T::ROWB + rl * 16), kx);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) kx[j] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float2 s2 = fmul2(qv[g][0], kx[0]);
#pragma unroll
          for (int j = 1; j < 4; ++j) s2 = ffma2(qv[g][j], kx[j], s2);
          v[u * G + g] = s2.x + s2.y;
        }
      }
      // ---- recursive-halving reduce across the LPR lanes of the row group -----------
#pragma unroll
      for (int st = 0, S = T::KP; st < T::HS; ++st, S >>= 1) {
        const int o = (T::LPR >> 1) >> st;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < S / 2; ++j) {
          const float send = up ? v[j] : v[j + S / 2];
          const float keep = up ? v[j + S / 2] : v[j];
          v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
#pragma unroll
      for (int o = T::REP >> 1; o >= 1; o >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
      const int hb = (rl / T::REP) * T::CNT;
      const bool writer = (rl % T::REP) == 0;
#pragma unroll
      for (int k = 0; k < T::CNT; ++k) {
        const int idx = hb + k;
        if (writer && idx < T::K) {
          const int u = idx / G, g = idx % G;
          const int t = u * T::RPW + rg;
          const int i = tb + t;
          const float sv = (i < end) ? v[k] : -INFINITY;
          sS[g * T::TT + t] = sv;
          if (i < end) scoreg[(size_t)g * d.sld + i] = sv;
        }
      }
      __syncwarp();
      // ---- tile max, rescale factors --------------------------------------------------
      float corr[G], mn[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float tm = -INFINITY;
#pragma unroll
        for (int t = 0; t < T::TT; t += 4) {
          const float4 s4 = *reinterpret_cast<const float4*>(&sS[g * T::TT + t]);
          tm = fmaxf(tm, fmaxf(fmaxf(s4.x, s4.y), fmaxf(s4.z, s4.w)));
        }
        mn[g] = fmaxf(m[g], tm);
        corr[g] = (m[g] == mn[g]) ? 1.f : expf(m[g] - mn[g]);
        zp[g] *= corr[g];
      }
      // ---- probabilities, once per (token, head) by its holder lane ------------------
#pragma unroll
      for (int k = 0; k < T::CNT; ++k) {
        const int idx = hb + k;
        if (writer && idx < T::K) {
          const int u = idx / G, g = idx % G;
          const int t = u * T::RPW + rg;
          const float sv = sS[g * T::TT + t];
          // register arrays must stay statically indexed (a runtime g would spill them)
          float mg = mn[0];
#pragma unroll
          for (int gg = 1; gg < G; ++gg) mg = (g == gg) ? mn[gg] : mg;
          const float p = (sv == -INFINITY) ? 0.f : expf(sv - mg);
          sP[g * T::TT + t] = p;
#pragma unroll
          for (int gg = 0; gg < G; ++gg) zp[gg] += (g == gg) ? p : 0.f;
        }
      }
      __syncwarp();
      // ---- P.V ------------------------------------------------------------------------
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (corr[g] != 1.f) {
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[g][j] = fmul2(acc[g][j], make_float2(corr[g], corr[g]));
        }
        m[g] = mn[g];
      }
#pragma unroll
      for (int u = 0; u < T::U; ++u) {
        const int t = u * T::RPW + rg;
        const int r = rb + t;
        const int tok = tb + t;
        if (tok >= end) continue;
        float2 vx[4];
        if (tok < n8) {
          code8_to_f2(*reinterpret_cast<const uint2*>(stV + (r & ~3) * T::ROWB + (r & 3) * D + rl * 8), vx);
          load_scales(sc, d, c, h, s_seg[tok - begin], D, rl);
#pragma unroll
          for (int j = 0; j < 4; ++j) vx[j] = fmul2(vx[j], sc.v[j]);
        } else {
          half8_to_f2(*reinterpret_cast<const uint4*>(stV + r * T::ROWB + rl * 16), vx);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float p = sP[g * T::TT + t];
          const float2 p2 = make_float2(p, p);
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[g][j] = ffma2(p2, vx[j], acc[g][j]);
        }
      }
      __syncwarp();   // stage rows and sS/sP are reused after this
      if (lane == 0) mbar_arrive(sbase + T::OFF_BAR + 8 * (kStages + s));
    }

    // ---- reduce acc across row groups; z across the warp -------------------------------
#pragma unroll
    for (int o = T::LPR; o < 32; o <<= 1) {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[g][j].x += __shfl_xor_sync(0xffffffffu, acc[g][j].x, o);
          acc[g][j].y += __shfl_xor_sync(0xffffffffu, acc[g][j].y, o);
        }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) zp[g] += __shfl_xor_sync(0xffffffffu, zp[g], o);
    // stash (m, z, acc) per warp; aliases the stage ring, idle once every consumer
    // has passed its last stage (named barrier over the consumer warps only)
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32));
    float* wacc = reinterpret_cast<float*>(smem);                 // [warps][G][D]
    float* wm = wacc + kConsumerWarps * G * D;                    // [warps][G]
    float* wz = wm + kConsumerWarps * G;
    if (lane < T::LPR) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          wacc[(warp * G + g) * D + rl * 8 + 2 * j] = acc[g][j].x;
          wacc[(warp * G + g) * D + rl * 8 + 2 * j + 1] = acc[g][j].y;
        }
      }
    }
    if (lane == 0) {
#pragma unroll
      for (int g = 0; g < G; ++g) { wm[warp * G + g] = m[g]; wz[warp * G + g] = zp[g]; }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32));
    const size_t pbase = ((size_t)c * Hq + (size_t)h * G) * d.npart + 2 * split;   // whole split: slot 2s
    for (int idx = threadIdx.x; idx < G * D; idx += kConsumerWarps * 32) {
      const int g = idx / D, dd = idx % D;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, wm[w * G + g]);
      float O = 0.f, Z = 0.f;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        const float mw = wm[w * G + g];
        if (mw == -INFINITY) continue;
        const float f = expf(mw - M);
        O += f * wacc[(w * G + g) * D + dd];
        Z += f * wz[w * G + g];
      }
      const size_t pi = pbase + (size_t)g * d.npart;
      d.po[pi * D + dd] = O;
      if (dd == 0) { d.pm[pi] = M; d.pz[pi] = Z; }
    }
  }
}

// ============================================================================================
// Tensor-core path (head_dim 64 / 128): both q.K^T and P.V on mma.sync.m16n8k16.
//
// Staging: each of the CTA's 4 warps owns a private ring (RING bytes) of tile slots, 16
// entries per tile, and fills it with 128B-swizzled TMA gathers (gather4 through the *_sw
// tensor maps: chunk j of 128-byte line L sits at j ^ (L & 7)), so TMA issue is spread over
// the warps and no warp waits on another. A split that is entirely INT8 uses half-size
// slots and gets twice the pipeline depth.
//
// q.K^T: entries = M, GQA heads = N (<= 8), head dims = K, under a fixed head-dim
// permutation (k-indices {2c,2c+1,2c+8,2c+9} of k-step kk are dims 16kk+4c+{0..3}) so each
// thread's A fragment is one contiguous, conflict-free smem word.
//   FP16 entries: A = K (exact), B = q (exact).
//   INT8 entries of one segment: A = codes (exact in fp16), B = q*k_scale*2^7 split into fp16
//     hi + lo (two MMAs, ~2^-22 relative) -> the reference's sum_d q_d (code_d scale_d).
//   Mixed tiles: A = dequantised K (fp32) split hi/lo, B = q.
// P.V: O^T[dims x heads] += V^T[dims x entries] P^T[entries x heads]. Entries are permuted
// (k-indices {2c,2c+1,2c+8,2c+9} = entries 4c..4c+3) and output dims too (thread g owns the
// contiguous slice [DS*g, DS*g+DS), DS = D/8, dim(mt, g, half) = DS*g + 2mt + half), so A
// fragments are PRMT-paired from contiguous 16/32-byte smem slices. P is split hi/lo in
// fp16 (two MMAs). INT8 tiles of one segment multiply codes (exact) and apply the segment's
// fp32 V scale per output element after each m-tile's MMA; mixed tiles dequantise in fp32
// and split hi/lo. The accumulator columns a thread owns are exactly the two heads whose
// running max it tracks, so the online-softmax rescale needs no data exchange.
constexpr int kMmaWarps = 4;

// Debug build (-DCKV_TRACE): %globaltimer stamps at the tcgen05 path's phase boundaries for the
// first kTraceCtas CTAs of the last launch, read back with ckv_debug_trace().
#ifdef CKV_TRACE
constexpr int kTraceCtas = 32768;
__device__ unsigned long long g_trace[kTraceCtas][16];
__device__ __forceinline__ void stamp(int i) {
  const unsigned b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0 && b < kTraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[b][i] = t;
    if (i == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_trace[b][15] = sm;
    }
  }
}
#define CKV_STAMP(i) stamp(i)
// persistent tcgen05 kernel: clock64 per item (first 64 items of each CTA), 12 events
constexpr int kPtCtas = 512, kPtItems = 64;
__device__ long long g_ptrace[kPtCtas][kPtItems][12];
#define CKV_PSTAMP(j, i)                                                      \
  do {                                                                        \
    if ((j) < kPtItems && blockIdx.x < kPtCtas) g_ptrace[blockIdx.x][(j)][(i)] = clock64(); \
  } while (0)
// step timeline (tools/trace_timeline.py): %globaltimer at CTA start / end + SM id per kernel
// kind (0 general split, 1 persistent tcgen05, 2 combine, 3 FP16 stream), read back with ckv_debug_timeline()
constexpr int kTlCtas = 8192;
__device__ unsigned long long g_tl[4][kTlCtas][4];
__device__ __forceinline__ void tl_stamp(int kind, int ev) {
  const unsigned b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0 && b < kTlCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tl[kind][b][ev] = t;
    if (ev == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_tl[kind][b][3] = sm;
    }
  }
}
#define CKV_TL(kind, ev) tl_stamp(kind, ev)
#else
#define CKV_PSTAMP(j, i)
#define CKV_TL(kind, ev)
#endif
#ifndef CKV_NO_TC
constexpr bool kTcEnabled = true;    // tcgen05 path for single-segment INT8 splits (D = 128)
#else
constexpr bool kTcEnabled = false;
#endif

template <int D, int G>
struct TrM {
  static constexpr int TT = 16;                        // entries per tile (one MMA M block)
  static constexpr int NSUB = D / 64;                  // 128-byte lines per fp16 row
  static constexpr int SUB = TT * 128;                 // 16 lines = 2 KB, 1024-aligned
  static constexpr int SLOT16 = 2 * NSUB * SUB;        // K and V, FP16 capacity
  static constexpr int SLOT8 = 2 * SUB;                // K and V, INT8 only
  static constexpr int RING = 16384;                   // per warp
  static constexpr int STAGES16 = RING / SLOT16;
  static constexpr int STAGES8 = RING / SLOT8 > 6 ? 6 : RING / SLOT8;
  static constexpr int KSTEPS = D / 16;
  static constexpr int MT = D / 16;                    // P.V m-tiles
  static constexpr int DS = D / 8;                     // dims per thread slice
  static constexpr int OFF_BAR = kMmaWarps * RING;
  static constexpr int OFF_ROW = OFF_BAR + kMmaWarps * 8 * 8;
  static constexpr int OFF_SEG = OFF_ROW + (kSplitTokens + kAbsorbTokens) * 4;
  static constexpr int OFF_P = OFF_SEG + (kSplitTokens + kAbsorbTokens) * 4;   // [warps][hi/lo][8 heads][16] fp16
  static constexpr int OFF_X = OFF_P + kMmaWarps * 2 * 8 * TT * 2;   // tcgen05 path: max / sum exchange
  static constexpr int SMEM = OFF_X + 1024;   // tcgen05 exchange / general-kernel split list
  static constexpr int KS8 = D / 32;                   // IMMA k-steps over head dims
  // integer path: 4 ring slots of 2 KB + per-warp scores [G][128] fp32 + max [8] in the same ring
  static constexpr int R8_SLOTS = 4;
  static constexpr int R8_S = R8_SLOTS * TT * 128;
  static_assert(R8_S + G * (kSplitTokens / kMmaWarps) * 4 + 8 * 4 <= RING, "integer-path ring layout");
  static_assert(kMmaWarps * G * (D + 2) * 4 <= kMmaWarps * RING, "epilogue alias");
  static_assert(G <= 8, "heads map to the MMA N dimension");
};

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tma_tile_row(uint32_t dst, const CUtensorMap* map, int col, int row, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(bar) : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
// D(s32) += A(s8, 16x32 row) x B(8-bit digit, 32x8 col); BT = "s8" or "u8"
__device__ __forceinline__ void imma_s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void imma_u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                        uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 16x16 int8 block, transposed: lane (g, c) gets rows 4c..4c+3 of columns g and g+8.
__device__ __forceinline__ void ldsm_b8_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m16n16.x1.trans.shared.b8 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ __half2 h2_1152() { return __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480)); }
// 4 int8 codes -> two half2 holding the exact code values (1024 + biased byte - 1152).
__device__ __forceinline__ void codes4_to_h2(uint32_t w, uint32_t& lo, uint32_t& hi) {
  const uint32_t b = w ^ 0x80808080u;
  uint32_t x = __byte_perm(b, 0x64646464u, 0x5140), y = __byte_perm(b, 0x64646464u, 0x5342);
  __half2 hx = __hsub2(*reinterpret_cast<__half2*>(&x), h2_1152()), hy = __hsub2(*reinterpret_cast<__half2*>(&y), h2_1152());
  lo = *reinterpret_cast<uint32_t*>(&hx);
  hi = *reinterpret_cast<uint32_t*>(&hy);
}
// byte k of biased word a and byte k of biased word b -> half2 (exact code values)
__device__ __forceinline__ uint32_t pair_codes(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t x = (__byte_perm(a, b, sel) & 0x00FF00FFu) | 0x64006400u;
  __half2 h = __hsub2(*reinterpret_cast<__half2*>(&x), h2_1152());
  return *reinterpret_cast<uint32_t*>(&h);
}
// fp32 pair -> (hi, lo) fp16 pairs with hi + lo = x to ~2^-22.
__device__ __forceinline__ void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ float h2lo(uint32_t w) { return __low2float(*reinterpret_cast<const __half2*>(&w)); }
__device__ __forceinline__ float h2hi(uint32_t w) { return __high2float(*reinterpret_cast<const __half2*>(&w)); }

// Stage tile `k` (entries [16k, 16k + 16) of the split) into a slot: gather4 per 4 entries
// of one type, single-row tiles at the INT8/FP16 boundary and the split's tail. Called by the
// whole warp with warp-uniform arguments; one elected lane issues, so every TMA operand
// lives in uniform registers (no per-lane waterfall).
template <int D, int G>
__device__ __forceinline__ void issue_tile(const Maps& maps, const int* s_row, int k, int ntok, int begin,
                                           int n8, uint32_t slot, uint32_t vofs, uint32_t bar) {
  using T = TrM<D, G>;
  const int j = k * T::TT;
  const int nrow = min(T::TT, ntok - j);
  const int n8s = max(0, min(nrow, n8 - (begin + j)));
  const bool leader = elect_one();
  if (leader) mbar_arrive_tx(bar, (uint32_t)(n8s * 2 * D + (nrow - n8s) * 4 * D));
  const uint32_t kb = slot, vb = slot + vofs;
  for (int g0 = 0; g0 < nrow; g0 += 4) {
    if (g0 + 4 <= nrow && (g0 + 4 <= n8s || g0 >= n8s)) {
      const int4 r = *reinterpret_cast<const int4*>(s_row + j + g0);
      if (g0 >= n8s) {
#pragma unroll
        for (int sub = 0; sub < T::NSUB; ++sub) {
          if (leader) {
            tma_gather4(kb + sub * T::SUB + g0 * 128, &maps.kf_sw, r.x, r.y, r.z, r.w, bar, sub * 64);
            tma_gather4(vb + sub * T::SUB + g0 * 128, &maps.vf_sw, r.x, r.y, r.z, r.w, bar, sub * 64);
          }
        }
      } else if (leader) {
        tma_gather4(kb + g0 * 128, &maps.kq_sw, r.x, r.y, r.z, r.w, bar, 0);
        tma_gather4(vb + g0 * 128, &maps.vq_sw, r.x, r.y, r.z, r.w, bar, 0);
      }
    } else {
      for (int r = g0; r < min(g0 + 4, nrow); ++r) {
        const int rr = s_row[j + r];
        if (!leader) continue;
        if (r < n8s) {
          tma_tile_row(kb + r * 128, &maps.kq_sw, 0, rr, bar);
          tma_tile_row(vb + r * 128, &maps.vq_sw, 0, rr, bar);
        } else {
#pragma unroll
          for (int sub = 0; sub < T::NSUB; ++sub) {
            tma_tile_row(kb + sub * T::SUB + r * 128, &maps.kf_sw, sub * 64, rr, bar);
            tma_tile_row(vb + sub * T::SUB + r * 128, &maps.vf_sw, sub * 64, rr, bar);
          }
        }
      }
    }
  }
}

// Integer path: stage one 16-entry tile of INT8 K (or V) rows only, one 128-byte line each.
template <int D, int G>
__device__ __forceinline__ void issue_tile8(const Maps& maps, const int* s_row, int k, int ntok, bool vside,
                                            uint32_t slot, uint32_t bar) {
  using T = TrM<D, G>;
  const int j = k * T::TT;
  const int nrow = min(T::TT, ntok - j);
  const bool leader = elect_one();
  if (leader) mbar_arrive_tx(bar, (uint32_t)(nrow * D));
  const CUtensorMap* m = vside ? &maps.vq_sw : &maps.kq_sw;
  for (int g0 = 0; g0 < nrow; g0 += 4) {
    if (g0 + 4 <= nrow) {
      const int4 r = *reinterpret_cast<const int4*>(s_row + j + g0);
      if (leader) tma_gather4(slot + g0 * 128, m, r.x, r.y, r.z, r.w, bar, 0);
    } else {
      for (int r = g0; r < nrow; ++r) {
        const int rr = s_row[j + r];
        if (leader) tma_tile_row(slot + r * 128, m, 0, rr, bar);
      }
    }
  }
}

// smem address of the 16-byte chunk holding dims [dim0, dim0+8) of an FP16 row, or bytes
// [byte0, byte0+16) of an INT8 row (both in the row's 128-byte lines, swizzled).
template <int D>
__device__ __forceinline__ uint32_t fp16_chunk(uint32_t base, int row, int dim0) {
  const uint32_t byte = 2u * dim0;
  return base + (byte >> 7) * (16 * 128) + row * 128 + ((((byte >> 4) & 7) ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint32_t int8_chunk(uint32_t base, int row, int byte0) {
  return base + row * 128 + ((((uint32_t)byte0 >> 4) ^ (row & 7)) << 4) + (byte0 & 15);
}

// Merge the 4 warps' (m, z, O) of one (cache, KV head, split) into the split partials.
template <int D, int G>
__device__ __forceinline__ void merge_warps(const Dev& d, int c, int h, int split, const float* wacc,
                                            const float* wm, const float* wz) {
  const size_t pbase = ((size_t)c * d.Hq + (size_t)h * G) * d.npart + split;   // split = partial slot
  for (int idx = threadIdx.x; idx < G * D; idx += kMmaWarps * 32) {
    const int g = idx / D, dd = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) M = fmaxf(M, wm[w * G + g]);
    float Ov = 0.f, Z = 0.f;
#pragma unroll
    for (int w = 0; w < kMmaWarps; ++w) {
      const float mw = wm[w * G + g];
      if (mw == -INFINITY) continue;
      const float f = expf(mw - M);
      Ov += f * wacc[(w * G + g) * D + dd];
      Z += f * wz[w * G + g];
    }
    const size_t pi = pbase + (size_t)g * d.npart;
    d.po[pi * D + dd] = Ov;
    if (dd == 0) { d.pm[pi] = M; d.pz[pi] = Z; }
  }
}

// ============================================================================================
// INT8 split of one segment: integer tensor cores on the raw codes.
//   pass 1 (K): S = codes . q', q' = q * k_scale * 2^E as three byte digits (s8 hi, u8 mid/lo),
//     three IMMA m16n8k32 per 32 dims, exact int32, combined in fp32 -> scores to smem + the
//     EMA scratch; the warp's max per head is then known, so no online rescaling is needed.
//   pass 2 (V): P = exp(s - max) as 24-bit fixed point (three u8 digits); V^T fragments come
//     straight from ldmatrix.m16n16.trans.b8 (LDSM.8.MT1616); three IMMA per 16 dims accumulate
//     exact int32 over the whole split; one conversion x the segment's V scale at the end.
// Loads run through a 4-slot ring per warp as one sequence K_0..K_{n-1}, V_0..V_{n-1}; the other
// half of the warp's ring holds its scores.
template <int D, int G>
__device__ __forceinline__ void issue_seq8(const Maps& maps, const int* s_row, int e, int nmine, int warp,
                                           int ntok, uint32_t ring, uint32_t bars) {
  using T = TrM<D, G>;
  if (e >= 2 * nmine) return;
  const int i = e < nmine ? e : e - nmine;
  issue_tile8<D, G>(maps, s_row, warp + kMmaWarps * i, ntok, e >= nmine, ring + (e % T::R8_SLOTS) * (T::TT * 128),
                    bars + 8 * (e % T::R8_SLOTS));
}

template <int D, int G>
__device__ __forceinline__ void attend_int8_split(const Dev& d, const Maps& maps, int c, int c0, int h, int split,
                                                  int begin, int end, int ntok, int ntiles, int warp, int lane,
                                                  const __half* __restrict__ q, float qscale, const int* s_row,
                                                  int sg, uint8_t* smem, uint32_t sbase) {
  using T = TrM<D, G>;
  constexpr int SLOT = T::TT * 128;
  const uint32_t ring = sbase + warp * T::RING;
  const uint32_t bars = sbase + T::OFF_BAR + 8 * warp * 8;
  const int nmine = ntiles > warp ? (ntiles - warp + kMmaWarps - 1) / kMmaWarps : 0;   // <= 8
  for (int e = 0; e < T::R8_SLOTS; ++e) issue_seq8<D, G>(maps, s_row, e, nmine, warp, ntok, ring, bars);

  const int Hq = d.Hq;
  const int gq = lane >> 2, cq = lane & 3;
  const int hA = 2 * cq, hB = 2 * cq + 1;
  const bool realA = hA < G, realB = hB < G;
  float* sS = reinterpret_cast<float*>(smem + warp * T::RING + T::R8_S);          // [G][128]
  float* sM = sS + G * (kSplitTokens / kMmaWarps);                                // [8]
  float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.sld;
  const size_t soff = (((size_t)c * d.smax + sg) * d.Hkv + h) * D;

  // ---- q' = q * k_scale as 24-bit fixed point, three byte digits per B fragment --------------
  uint32_t qd[3][T::KS8][2];
  float sfix;
  {
    float qv[T::KS8][2][4];
    float mx = 0.f;
    const __half* qp = q + ((size_t)(c - c0) * Hq + (size_t)h * G + gq) * D;
#pragma unroll
    for (int ks = 0; ks < T::KS8; ++ks)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        const int d0 = 32 * ks + 16 * hf + 4 * cq;
        const float4 k4 = __ldg(reinterpret_cast<const float4*>(d.ksc + soff + d0));
        float2 q01 = make_float2(0.f, 0.f), q23 = q01;
        if (gq < G) {
          const uint2 w = *reinterpret_cast<const uint2*>(qp + d0);
          q01 = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
          q23 = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
        }
        qv[ks][hf][0] = q01.x * k4.x; qv[ks][hf][1] = q01.y * k4.y;
        qv[ks][hf][2] = q23.x * k4.z; qv[ks][hf][3] = q23.y * k4.w;
#pragma unroll
        for (int e = 0; e < 4; ++e) mx = fmaxf(mx, fabsf(qv[ks][hf][e]));
      }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int ex = 0;
    if (mx > 0.f) frexpf(mx, &ex);          // mx = f * 2^ex, f in [0.5, 1)
    const int E = 23 - ex;                  // |q' * 2^E| < 2^23
    const float up = ldexpf(1.f, E);
    sfix = qscale * ldexpf(1.f, -E);
#pragma unroll
    for (int ks = 0; ks < T::KS8; ++ks)
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int v = __float2int_rn(qv[ks][hf][e] * up);
          w0 |= (uint32_t)(v & 255) << (8 * e);
          w1 |= (uint32_t)((v >> 8) & 255) << (8 * e);
          w2 |= (uint32_t)((v >> 16) & 255) << (8 * e);
        }
        qd[0][ks][hf] = w0; qd[1][ks][hf] = w1; qd[2][ks][hf] = w2;
      }
  }

  // ---- pass 1: scores ----------------------------------------------------------------------
  // rows gq and gq+8 share the swizzle phase (gq & 7): one base offset per row, chunk XOR per k-step
  const uint32_t kro0 = gq * 128 + 4 * cq, kro1 = kro0 + 8 * 128, ksw = (uint32_t)(gq & 7) << 4;
  float* scA = scoreg + (size_t)hA * d.sld + begin + gq;   // + tile offset
  float* scB = scoreg + (size_t)hB * d.sld + begin + gq;
  float mA = -INFINITY, mB = -INFINITY;
  for (int i = 0; i < nmine; ++i) {
    const int k = warp + kMmaWarps * i;
    const uint32_t slot = ring + (i % T::R8_SLOTS) * SLOT;
    mbar_wait(bars + 8 * (i % T::R8_SLOTS), (i / T::R8_SLOTS) & 1);
    const int tb = begin + k * T::TT;
    const int nvalid = min(T::TT, end - tb);
    int acc[3][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
    for (int ks = 0; ks < T::KS8; ++ks) {
      const uint32_t c0o = ((uint32_t)(2 * ks) << 4) ^ ksw, c1o = ((uint32_t)(2 * ks + 1) << 4) ^ ksw;
      const uint32_t a0 = lds32(slot + kro0 + c0o);
      const uint32_t a1 = lds32(slot + kro1 + c0o);
      const uint32_t a2 = lds32(slot + kro0 + c1o);
      const uint32_t a3 = lds32(slot + kro1 + c1o);
      imma_u8(acc[0], a0, a1, a2, a3, qd[0][ks][0], qd[0][ks][1]);
      imma_u8(acc[1], a0, a1, a2, a3, qd[1][ks][0], qd[1][ks][1]);
      imma_s8(acc[2], a0, a1, a2, a3, qd[2][ks][0], qd[2][ks][1]);
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue_seq8<D, G>(maps, s_row, i + T::R8_SLOTS, nmine, warp, ntok, ring, bars);
    float sv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      sv[e] = fmaf((float)acc[2][e], 65536.f, fmaf((float)acc[1][e], 256.f, (float)acc[0][e])) * sfix;
    const bool v0 = gq < nvalid, v1 = gq + 8 < nvalid;
    const float s0 = v0 ? sv[0] : -INFINITY, s1 = v0 ? sv[1] : -INFINITY;
    const float s2 = v1 ? sv[2] : -INFINITY, s3 = v1 ? sv[3] : -INFINITY;
    const int tl = i * T::TT;   // this tile's column in the warp's score buffer
    const int to = k * T::TT;   // tile offset inside the split
    if (realA) {
      sS[hA * 128 + tl + gq] = s0; sS[hA * 128 + tl + gq + 8] = s2;
      if (v0) scA[to] = s0;
      if (v1) scA[to + 8] = s2;
    }
    if (realB) {
      sS[hB * 128 + tl + gq] = s1; sS[hB * 128 + tl + gq + 8] = s3;
      if (v0) scB[to] = s1;
      if (v1) scB[to + 8] = s3;
    }
    mA = fmaxf(mA, fmaxf(s0, s2));
    mB = fmaxf(mB, fmaxf(s1, s3));
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    mA = fmaxf(mA, __shfl_xor_sync(0xffffffffu, mA, o));
    mB = fmaxf(mB, __shfl_xor_sync(0xffffffffu, mB, o));
  }
  if (gq == 0) {
    if (realA) sM[hA] = mA;
    if (realB) sM[hB] = mB;
  }
  __syncwarp();
  const float Mg = gq < G ? sM[gq] : 0.f;

  // ---- pass 2: P (24-bit fixed point) . V, exact int32 over the split ---------------------------
  int O[3][T::MT][4];
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int mt = 0; mt < T::MT; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e) O[j][mt][e] = 0;
  long long zq = 0;
  const uint32_t vro = (uint32_t)(lane & 15) * 128, vsw = (uint32_t)(lane & 7) << 4;
  for (int i = 0; i < nmine; ++i) {
    const int e = nmine + i;                       // position in the load sequence
    const uint32_t slot = ring + (e % T::R8_SLOTS) * SLOT;
    uint32_t pd0 = 0, pd1 = 0, pd2 = 0;
    if (gq < G && Mg != -INFINITY) {
      const float4 s4 = *reinterpret_cast<const float4*>(sS + gq * 128 + i * T::TT + 4 * cq);
      const float sj[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t v = sj[e] == -INFINITY ? 0u : (uint32_t)__float2int_rn(expf(sj[e] - Mg) * 8388608.f);
        zq += v;
        pd0 |= (v & 255u) << (8 * e);
        pd1 |= ((v >> 8) & 255u) << (8 * e);
        pd2 |= ((v >> 16) & 255u) << (8 * e);
      }
    }
    mbar_wait(bars + 8 * (e % T::R8_SLOTS), (e / T::R8_SLOTS) & 1);
    const uint32_t vrow = slot + vro;
#pragma unroll
    for (int mt = 0; mt < T::MT; ++mt) {
      uint32_t a0, a1;
      ldsm_b8_t(vrow + (((uint32_t)mt << 4) ^ vsw), a0, a1);
      imma_u8(O[0][mt], a0, a1, 0u, 0u, pd0, 0u);
      imma_u8(O[1][mt], a0, a1, 0u, 0u, pd1, 0u);
      imma_u8(O[2][mt], a0, a1, 0u, 0u, pd2, 0u);
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue_seq8<D, G>(maps, s_row, e + T::R8_SLOTS, nmine, warp, ntok, ring, bars);
  }
  // z per head: lanes (g, *) hold head g's partial sums over their entries
  zq += __shfl_xor_sync(0xffffffffu, zq, 1);
  zq += __shfl_xor_sync(0xffffffffu, zq, 2);
  __syncthreads();   // every warp is done with its ring: reuse it for the (m, z, O) stash
  float* wacc = reinterpret_cast<float*>(smem);
  float* wm = wacc + kMmaWarps * G * D;
  float* wz = wm + kMmaWarps * G;
  const float inv = 1.f / 8388608.f;
#pragma unroll
  for (int mt = 0; mt < T::MT; ++mt) {
    const int da = 16 * mt + gq, db = da + 8;
    const float va = __ldg(d.vsc + soff + da) * inv, vb = __ldg(d.vsc + soff + db) * inv;
    float o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = fmaf((float)O[2][mt][e], 65536.f, fmaf((float)O[1][mt][e], 256.f, (float)O[0][mt][e]));
    if (realA) {
      wacc[(warp * G + hA) * D + da] = o[0] * va;
      wacc[(warp * G + hA) * D + db] = o[2] * vb;
    }
    if (realB) {
      wacc[(warp * G + hB) * D + da] = o[1] * va;
      wacc[(warp * G + hB) * D + db] = o[3] * vb;
    }
  }
  if (gq == 0) {
    if (realA) wm[warp * G + hA] = mA;
    if (realB) wm[warp * G + hB] = mB;
  }
  if (cq == 0 && gq < G) wz[warp * G + gq] = (float)zq * inv;
  __syncthreads();
  merge_warps<D, G>(d, c, h, split, wacc, wm, wz);
}



// ============================================================================================
// Persistent tcgen05 kernel for single-segment INT8 splits (D = 128): "bulk" splits whose
// entries are all read as codes of one segment. Each CTA walks its share of the (cache, KV
// head, split) items; roles are warp-specialised so the next item's loads stream while the
// current item's epilogue runs:
//   warp 0     producer: bulk test, row coordinates (slot -> TMA row), then per item the chunk
//              sequence K_0..K_{n-1}, V_0..V_{n-1} (128 entries = 16 KB each, 32 TMA gather4)
//              into a SLOTS-deep ring.
//   warp 1     MMA issuer (one lane): QK  S[128 x N] = K_c (s8, SW128 K-major) . Qd (s8 digits),
//              PV  O[128 dims x N] = V_c^T (s8, SW128 read MN-major) . Pd (u8 digits); exact
//              int32 in TMEM, double-buffered across items.
//   warps 2-5  epilogue (TMEM lane quadrant = warp % 4): Qd = q * k_scale * 2^E_h as three
//              balanced signed byte digits; scores (EMA scratch); split max; P = exp(s - m) as
//              24-bit fixed point in three u8 digits; O x V scale -> split partials.
// Barrier phases: per-item barriers complete exactly once per item (chunks past the item's end
// get empty commits / arrivals), so their parity is the item counter's; per-buffer barriers
// complete once per two items.
template <int G>
struct TcP {
  static constexpr int N = 3 * G <= 16 ? 16 : 32;    // MMA N: G heads x 3 digits (n = j*G + h)
  static constexpr int SLOTS = N == 16 ? 6 : 5;
  static constexpr int SLOTB = 128 * 128;            // 128 entries x 128 B
  static constexpr int SCOLS = 4 * N;                // TMEM columns per item (O reuses chunk 0)
  static constexpr int NC = 2 * SCOLS <= 128 ? 128 : 256;
  static constexpr int QDB = N * 128;
  static constexpr int PCH = 128 * N;
  static constexpr int PB = 2;
  static constexpr int OFF_QD = SLOTS * SLOTB;
  static constexpr int OFF_PD = OFF_QD + 2 * QDB;
  static constexpr int OFF_ROW = OFF_PD + PB * PCH;   // [2][512] row coordinates (producer)
  static constexpr int OFF_ITEM = OFF_ROW + 2 * kSplitTokens * 4;   // [2] int4 item descriptors
  static constexpr int OFF_BAR = OFF_ITEM + 64;
  // barrier indices
  static constexpr int B_FULL = 0, B_EMPTY = SLOTS, B_IFULL = 2 * SLOTS, B_IEMPTY = B_IFULL + 2,
                       B_QD = B_IEMPTY + 2, B_SDONE = B_QD + 2, B_PRDY = B_SDONE + 4, B_PV = B_PRDY + 4,
                       B_O = B_PV + 4, B_TFREE = B_O + 1, N_BAR = B_TFREE + 2;
  static constexpr int OFF_X = OFF_BAR + 8 * N_BAR;   // sfix[2][8] f32, red[4][8] f32, zred[4][8] u64, tmem addr
  static constexpr int SMEM = OFF_X + 64 + 128 + 256 + 16;
  static constexpr int THREADS = 192;
  static_assert(SMEM <= 113 * 1024, "two CTAs per SM");
};

__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int G>
__device__ __forceinline__ void tc_items(const Dev& d, const Maps& maps, int c0, int ccount, const __half* __restrict__ q,
                                         float qscale, uint8_t* smem) {
  using T = TcP<G>;
  constexpr int D = 128, N = T::N, S = T::SLOTS;
  constexpr uint32_t IQK = tc::idesc_i8(128, N, true, true, false, false);
  constexpr uint32_t IPV = tc::idesc_i8(128, N, true, false, true, true);
  const uint32_t sbase = smem_u32(smem);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t bars = sbase + T::OFF_BAR;
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  int4* s_item = reinterpret_cast<int4*>(smem + T::OFF_ITEM);
  float* sfix = reinterpret_cast<float*>(smem + T::OFF_X);                  // [2][8]
  float* red = sfix + 16;                                                   // [4][8]
  unsigned long long* zred = reinterpret_cast<unsigned long long*>(smem + T::OFF_X + 192);   // [4][8]
  uint32_t* s_tm = reinterpret_cast<uint32_t*>(smem + T::OFF_X + 448);

  if (threadIdx.x == 0) {
    for (int i = 0; i < T::N_BAR; ++i) {
      const bool many = (i >= T::B_QD && i < T::B_QD + 2) || (i >= T::B_PRDY && i < T::B_PRDY + 4) ||
                        (i >= T::B_TFREE && i < T::B_TFREE + 2);
      mbar_init(bar(i), many ? 128 : 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tc::alloc(smem_u32(s_tm), T::NC);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = *reinterpret_cast<volatile uint32_t*>(s_tm);
  const int Hq = d.Hq, Hkv = d.Hkv, nsp = d.live_splits, npt = d.npart;
  const int total = ccount * Hkv * nsp;

  if (warp == 0) {
    // ===================================== producer =====================================
    // Small launches (few items per CTA, e.g. one layer of a decode forward) claim items
    // dynamically (one atomic per item on d.work, reset by k2_combine; the next claim issued
    // before this item's loads), so CTAs placed late beside the general-split kernel's CTAs
    // take fewer items; big launches stride statically (32 items' descriptors loaded at
    // once, one per lane).
    // The item stream runs one item ahead: the next item's descriptor and its 512 slot indices
    // (16 per lane, in registers) are requested before this item's chunks are issued, so the
    // dependent slot-table round trip (~1.7 us per item when serial) overlaps the ring refills.
    const bool dyn = d.dyn_items;
    int j = 0, g = 0;
    int kq = 0;
    if (dyn && lane == 0) kq = atomicAdd(d.work, 1);
    int base = (int)blockIdx.x - 32 * (int)gridDim.x;
    unsigned m = 0;
    bool done = false;
    int c = 0, h = 0, sp = 0, n = 0, sg = 0;   // this lane's descriptor in the current batch
    auto next = [&](int& ic, int& ih, int& isp, int& in, int& isg) -> bool {
      while (!m) {
        if (done) return false;
        int k;
        if (dyn) {
          const int k0 = __shfl_sync(0xffffffffu, kq, 0);
          if (k0 >= total) { done = true; return false; }
          if (lane == 0) kq = atomicAdd(d.work, 1);
          k = lane == 0 ? k0 : total;
        } else {
          base += 32 * (int)gridDim.x;
          if (base >= total) { done = true; return false; }
          k = base + lane * (int)gridDim.x;
        }
        c = 0; h = 0; sp = 0; n = 0; sg = 0;
        bool isb = false;
        if (k < total) {
          sp = k % nsp;
          h = (k / nsp) % Hkv;
          c = c0 + k / (nsp * Hkv);
          int b, e;
          part_range(d, sp, 0, d.len[c], d.nq[c], b, e);   // the split's codes part
          n = e;
          if (b < e) {
            sg = __ldg(d.seg + (size_t)c * d.cap + b);
            isb = sg == __ldg(d.seg + (size_t)c * d.cap + e - 1);
          }
        }
        m = __ballot_sync(0xffffffffu, isb);
      }
      const int L = __ffs(m) - 1;
      m &= m - 1;
      ic = __shfl_sync(0xffffffffu, c, L); ih = __shfl_sync(0xffffffffu, h, L);
      isp = __shfl_sync(0xffffffffu, sp, L); in = __shfl_sync(0xffffffffu, n, L);
      isg = __shfl_sync(0xffffffffu, sg, L);
      return true;
    };
    constexpr int SPL = kSplitTokens / 32;   // slot indices per lane
    auto load_slots = [&](int (&sv)[SPL], int ic, int isp, int in) {
      const int begin = isp * kSplitTokens, ntok = min(in, begin + kSplitTokens) - begin;
      const int* sl = d.slot + (size_t)ic * d.cap + begin;
#pragma unroll
      for (int i = 0; i < SPL; ++i) sv[i] = __ldg(sl + min(lane + 32 * i, ntok - 1));   // rows past the end repeat the last entry
    };
    int ic = 0, ih = 0, isp = 0, in = 0, isg = 0;
    int sv[SPL];
    bool have = next(ic, ih, isp, in, isg);
    if (have) load_slots(sv, ic, isp, in);
    while (have) {
      const int begin = isp * kSplitTokens, ntok = min(in, begin + kSplitTokens) - begin;
      int nc = 0, nh = 0, nsp2 = 0, nn = 0, nsg = 0;
      int nv[SPL];
      const bool nhave = next(nc, nh, nsp2, nn, nsg);
      if (nhave) load_slots(nv, nc, nsp2, nn);
      const int b = j & 1;
      if (j >= 2) mbar_wait(bar(T::B_IEMPTY + b), ((j >> 1) - 1) & 1);
      if (lane == 0) CKV_PSTAMP(j, 0);
      int* rows = reinterpret_cast<int*>(smem + T::OFF_ROW) + b * kSplitTokens;
      const size_t cb = (size_t)ic * d.cap;
#pragma unroll
      for (int i = 0; i < SPL; ++i) rows[lane + 32 * i] = code_row(cb, sv[i], Hkv, ih);   // code slots
      if (lane == 0) s_item[b] = make_int4(ic, ih | ((2 * isp) << 8), begin | (ntok << 20), isg);
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(T::B_IFULL + b));
      if (lane == 0) CKV_PSTAMP(j, 1);
      const int nch = (ntok + 127) >> 7;
      for (int e = 0; e < 2 * nch; ++e, ++g) {
        const int s = g % S, u = g / S;
        if (u > 0) mbar_wait(bar(T::B_EMPTY + s), (u - 1) & 1);
        const CUtensorMap* mp = e < nch ? &maps.kq_sw : &maps.vq_sw;
        const int ch = e < nch ? e : e - nch;
        const uint32_t dst = sbase + (uint32_t)s * T::SLOTB;
        const int* cr = rows + ch * 128;
        const bool leader = elect_one();
        if (leader) mbar_arrive_tx(bar(T::B_FULL + s), T::SLOTB);
#pragma unroll 1
        for (int r0 = 0; r0 < 128; r0 += 32) {
          int4 rr[8];
#pragma unroll
          for (int gq = 0; gq < 8; ++gq) rr[gq] = *reinterpret_cast<const int4*>(cr + r0 + 4 * gq);
          if (leader) {
#pragma unroll
            for (int gq = 0; gq < 8; ++gq)
              tma_gather4(dst + (r0 + 4 * gq) * 128, mp, rr[gq].x, rr[gq].y, rr[gq].z, rr[gq].w,
                          bar(T::B_FULL + s), 0);
          }
        }
      }
      if (lane == 0) CKV_PSTAMP(j, 2);
      ++j;
      have = nhave;
      ic = nc; ih = nh; isp = nsp2; in = nn; isg = nsg;
#pragma unroll
      for (int i = 0; i < SPL; ++i) sv[i] = nv[i];
    }
    const int b = j & 1;   // end marker
    if (j >= 2) mbar_wait(bar(T::B_IEMPTY + b), ((j >> 1) - 1) & 1);
    if (lane == 0) {
      s_item[b] = make_int4(-1, 0, 0, 0);
      mbar_arrive(bar(T::B_IFULL + b));
    }
  } else if (warp == 1) {
    // ===================================== MMA issuer =====================================
    if (lane == 0) {
      int j = 0, g = 0;
      for (;;) {
        const int b = j & 1;
        mbar_wait(bar(T::B_IFULL + b), (j >> 1) & 1);
        const uint4 itu = lds128(smem_u32(s_item + b));
        const int4 it = make_int4((int)itu.x, (int)itu.y, (int)itu.z, (int)itu.w);
        if (it.x < 0) break;
        CKV_PSTAMP(j, 3);
        const int ntok = it.z >> 20;
        const int nch = (ntok + 127) >> 7;
        mbar_wait(bar(T::B_QD + b), (j >> 1) & 1);
        if (j >= 2) mbar_wait(bar(T::B_TFREE + b), ((j >> 1) - 1) & 1);
        CKV_PSTAMP(j, 4);
        tc::fence_after();
        const uint32_t tS = tm + (uint32_t)(b * T::SCOLS);
        const uint32_t qd = sbase + T::OFF_QD + b * T::QDB;
        for (int ch = 0; ch < 4; ++ch) {
          if (ch < nch) {
            const int s = g % S;
            mbar_wait(bar(T::B_FULL + s), (g / S) & 1);
            tc::fence_after();
            const uint32_t slot = sbase + (uint32_t)s * T::SLOTB;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_i8(tS + ch * N, tc::sdesc(slot + 32 * ks, 16, 1024, tc::kSW128),
                         tc::sdesc(qd + 256 * ks, 128, 1024, tc::kInterleave), IQK, ks > 0);
            tc::commit(bar(T::B_EMPTY + s));
            ++g;
          }
          tc::commit(bar(T::B_SDONE + ch));
        }
        CKV_PSTAMP(j, 5);
        for (int ch = 0; ch < 4; ++ch) {
          mbar_wait(bar(T::B_PRDY + ch), j & 1);
          if (ch < nch) {
            const int s = g % S;
            mbar_wait(bar(T::B_FULL + s), (g / S) & 1);
            tc::fence_after();
            const uint32_t slot = sbase + (uint32_t)s * T::SLOTB;
            const uint32_t pb = sbase + T::OFF_PD + (uint32_t)((ch % T::PB) * T::PCH);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_i8(tS, tc::sdesc(slot + 4096 * ks, 8192, 1024, tc::kSW128),
                         tc::sdesc(pb + 512 * ks, 128, 2048, tc::kInterleave), IPV, (ch | ks) > 0);
            tc::commit(bar(T::B_EMPTY + s));
            ++g;
          }
          tc::commit(bar(T::B_PV + ch));
        }
        tc::commit(bar(T::B_O));
        CKV_PSTAMP(j, 6);
        ++j;
      }
    }
    __syncwarp();
  } else {
    // ===================================== epilogue =====================================
    const int et = threadIdx.x - 64;            // 0..127
    const int quad = warp & 3;                  // TMEM lanes 32*quad..
    const uint32_t tlane = (uint32_t)(32 * quad) << 16;
    // Item j+1's Qd digits are built while item j's P.V runs (after its P digits are handed to
    // the MMA warp, before its O is read), so the MMA starts item j+1's q.K^T as soon as the
    // TMEM buffer frees instead of waiting a global q / k-scale round trip per item.
    auto read_item = [&](int jj) -> int4 {
      const int bb = jj & 1;
      mbar_wait(bar(T::B_IFULL + bb), (jj >> 1) & 1);
      const uint4 itu = lds128(smem_u32(s_item + bb));
      return make_int4((int)itu.x, (int)itu.y, (int)itu.z, (int)itu.w);
    };
    auto build_qd = [&](const int4& it, int b) {
      const int c = it.x, h = it.y & 255, sg = it.w;
      const size_t soff = (((size_t)c * d.smax + sg) * Hkv + h) * D;
      uint8_t* qdb = smem + T::OFF_QD + b * T::QDB;
      // ---- Qd: balanced signed byte digits of q' = q * k_scale * 2^E_h (one head per warp) ----
      const __half* qh = q + ((size_t)(c - c0) * Hq + (size_t)h * G) * D;
      for (int idx = et; idx < G * 32; idx += 128) {
        const int hh = idx >> 5, d0 = (idx & 31) * 4;
        const uint2 w = *reinterpret_cast<const uint2*>(qh + hh * D + d0);
        const float4 k4 = __ldg(reinterpret_cast<const float4*>(d.ksc + soff + d0));
        const float2 q01 = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
        const float2 q23 = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
        const float qv[4] = {q01.x * k4.x, q01.y * k4.y, q23.x * k4.z, q23.y * k4.w};
        float mx = fmaxf(fmaxf(fabsf(qv[0]), fabsf(qv[1])), fmaxf(fabsf(qv[2]), fabsf(qv[3])));
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int ex = 0;
        if (mx > 0.f) frexpf(mx, &ex);
        const int E = 22 - ex;                // |q' * 2^E| < 2^22: three balanced digits
        const float up = ldexpf(1.f, E);
        if (lane == 0) sfix[b * 8 + hh] = qscale * ldexpf(1.f, -E);
        uint32_t dw[3] = {0u, 0u, 0u};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int x = __float2int_rn(qv[e] * up);
          const int x0 = ((x + 128) & 255) - 128;
          const int x1r = (x - x0) >> 8;
          const int x1 = ((x1r + 128) & 255) - 128;
          const int x2 = (x1r - x1) >> 8;
          dw[0] |= (uint32_t)(x0 & 255) << (8 * e);
          dw[1] |= (uint32_t)(x1 & 255) << (8 * e);
          dw[2] |= (uint32_t)(x2 & 255) << (8 * e);
        }
#pragma unroll
        for (int jj = 0; jj < 3; ++jj) {
          const int nn = jj * G + hh;
          *reinterpret_cast<uint32_t*>(qdb + (nn >> 3) * 1024 + (d0 >> 4) * 128 + (nn & 7) * 16 + (d0 & 15)) = dw[jj];
        }
      }
      for (int i = et; i < (N - 3 * G) * 32; i += 128) {
        const int nn = 3 * G + (i >> 5), d0 = (i & 31) * 4;
        *reinterpret_cast<uint32_t*>(qdb + (nn >> 3) * 1024 + (d0 >> 4) * 128 + (nn & 7) * 16 + (d0 & 15)) = 0u;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(bar(T::B_QD + b));
    };
    int j = 0;
    int4 it = read_item(0);
    if (it.x >= 0) build_qd(it, 0);
    while (it.x >= 0) {
      const int b = j & 1;
      if (et == 0) CKV_PSTAMP(j, 7);
      const int c = it.x, h = it.y & 255, split = it.y >> 8;
      const int begin = it.z & ((1 << 20) - 1), ntok = it.z >> 20, sg = it.w;
      const int nch = (ntok + 127) >> 7;
      const size_t soff = (((size_t)c * d.smax + sg) * Hkv + h) * D;
      const float vs = __ldg(d.vsc + soff + 32 * quad + lane) * (1.f / 8388608.f);
      if (et == 0) CKV_PSTAMP(j, 8);
      named_bar(1, 128);                         // sfix visible to every epilogue thread

      // ---- scores: entry 32*quad + lane of each chunk ----
      float sv[4][G];
      float mx[G], sf[G];
#pragma unroll
      for (int hh = 0; hh < G; ++hh) { mx[hh] = -INFINITY; sf[hh] = sfix[b * 8 + hh]; }
      float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.sld + begin;
      const uint32_t tS = tm + tlane + (uint32_t)(b * T::SCOLS);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        if (ch < nch) {
          mbar_wait(bar(T::B_SDONE + ch), j & 1);
          tc::fence_after();
          int a[N];
          tc::ld16(tS + ch * N, *reinterpret_cast<int(*)[16]>(a));
          if constexpr (N == 32) tc::ld16(tS + ch * N + 16, *reinterpret_cast<int(*)[16]>(a + 16));
          tc::wait_ld();
          const int tok = ch * 128 + 32 * quad + lane;
          const bool valid = tok < ntok;
#pragma unroll
          for (int hh = 0; hh < G; ++hh) {
            const float sc = fmaf((float)a[2 * G + hh], 65536.f, fmaf((float)a[G + hh], 256.f, (float)a[hh])) * sf[hh];
            sv[ch][hh] = valid ? sc : -INFINITY;
            if (valid) scoreg[(size_t)hh * d.sld + tok] = sc;
            mx[hh] = fmaxf(mx[hh], sv[ch][hh]);
          }
        } else {
#pragma unroll
          for (int hh = 0; hh < G; ++hh) sv[ch][hh] = -INFINITY;
        }
      }
      const int ew = warp - 2;
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], o));
        if (lane == 0) red[ew * 8 + hh] = mx[hh];
      }
      tc::fence_before();
      named_bar(1, 128);
      if (et == 0) CKV_PSTAMP(j, 9);
      float M[G];
#pragma unroll
      for (int hh = 0; hh < G; ++hh) M[hh] = fmaxf(fmaxf(red[hh], red[8 + hh]), fmaxf(red[16 + hh], red[24 + hh]));

      // ---- P digits per chunk (entry-major rows of N bytes) ----
      unsigned long long zq[G];
#pragma unroll
      for (int hh = 0; hh < G; ++hh) zq[hh] = 0ull;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        if (ch < nch) {
          if (ch >= T::PB) mbar_wait(bar(T::B_PV + ch - T::PB), j & 1);
          uint32_t w[N / 4];
#pragma unroll
          for (int i = 0; i < N / 4; ++i) w[i] = 0u;
#pragma unroll
          for (int hh = 0; hh < G; ++hh) {
            const uint32_t v = sv[ch][hh] == -INFINITY ? 0u : (uint32_t)__float2int_rn(expf(sv[ch][hh] - M[hh]) * 8388608.f);
            zq[hh] += v;
            w[hh >> 2] |= (v & 255u) << (8 * (hh & 3));
            w[(G + hh) >> 2] |= ((v >> 8) & 255u) << (8 * ((G + hh) & 3));
            w[(2 * G + hh) >> 2] |= (v >> 16) << (8 * ((2 * G + hh) & 3));
          }
          uint8_t* row = smem + T::OFF_PD + (ch % T::PB) * T::PCH + (32 * quad + lane) * 16;
#pragma unroll
          for (int gq = 0; gq < N / 16; ++gq)
            *reinterpret_cast<uint4*>(row + gq * 2048) = make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        mbar_arrive(bar(T::B_PRDY + ch));
      }
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) zq[hh] += __shfl_xor_sync(0xffffffffu, zq[hh], o);
        if (lane == 0) zred[ew * 8 + hh] = zq[hh];
      }

      // ---- next item's Qd while this item's P.V runs ----
      const int4 itn = read_item(j + 1);
      if (itn.x >= 0) build_qd(itn, b ^ 1);

      // ---- O epilogue: thread = head dim 32*quad + lane ----
      mbar_wait(bar(T::B_O), j & 1);
      if (et == 0) CKV_PSTAMP(j, 10);
      tc::fence_after();
      int a[N];
      tc::ld16(tm + tlane + (uint32_t)(b * T::SCOLS), *reinterpret_cast<int(*)[16]>(a));
      if constexpr (N == 32) tc::ld16(tm + tlane + (uint32_t)(b * T::SCOLS) + 16, *reinterpret_cast<int(*)[16]>(a + 16));
      tc::wait_ld();
      tc::fence_before();
      mbar_arrive(bar(T::B_TFREE + b));
      const int dim = 32 * quad + lane;
      const size_t pbase = ((size_t)c * Hq + (size_t)h * G) * npt + split;   // split = partial slot 2s
#pragma unroll
      for (int hh = 0; hh < G; ++hh) {
        const float o = fmaf((float)a[2 * G + hh], 65536.f, fmaf((float)a[G + hh], 256.f, (float)a[hh]));
        d.po[(pbase + (size_t)hh * npt) * D + dim] = o * vs;
      }
      named_bar(1, 128);                         // zred complete
      if (et < G) {
        const unsigned long long z = zred[et] + zred[8 + et] + zred[16 + et] + zred[24 + et];
        const size_t pi = pbase + (size_t)et * npt;
        d.pm[pi] = fmaxf(fmaxf(red[et], red[8 + et]), fmaxf(red[16 + et], red[24 + et]));
        d.pz[pi] = (float)z * (1.f / 8388608.f);
      }
      named_bar(1, 128);                         // red / zred / s_item[b] free for reuse
      if (et == 0) mbar_arrive(bar(T::B_IEMPTY + b));
      if (et == 0) CKV_PSTAMP(j, 11);
      ++j;
      it = itn;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after();
    tc::dealloc(tm, T::NC);
  }
}

template <int G>
__global__ void __launch_bounds__(TcP<G>::THREADS, 2)
k2_i8_persistent(Dev d, const __grid_constant__ Maps maps, int c0, int ccount, const __half* __restrict__ q,
                 float qscale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // an inline K1 (this grid's programmatic dependent; it waits for this grid at its exit) runs
  // in the SM room beside our CTAs instead of after them
  asm volatile("griddepcontrol.launch_dependents;");
  CKV_TL(1, 0);
  tc_items<G>(d, maps, c0, ccount, q, qscale, smem);
  CKV_TL(1, 2);
  // Launched as a programmatic dependent of the general-split kernel (they share no data, so
  // this grid starts beside it): do not complete before that grid has, so the combine launched
  // after this kernel sees both kernels' partials. A no-op without a prerequisite grid.
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// One split of one (cache, KV head) on the 4-warp mma.sync path (FP16, mixed and multi-segment
// INT8 splits; single-segment INT8 splits too when the tcgen05 kernel is not used).
// BULK = false (the general kernel beside the tcgen05 grid, whose single-segment codes splits
// never reach it): the integer bulk path is compiled out (fewer registers, no spills).
template <int D, int G, bool BULK = true>
__device__ __forceinline__ void mma_split(const Dev& d, const Maps& maps, int c0, const __half* __restrict__ q,
                                          float qscale, int c, int h, int begin, int end, int split,
                                          uint8_t* smem, bool rows_staged = false) {
  // `split` is the partial slot the result goes to; [begin, end) the entries
  using T = TrM<D, G>;
  if (begin >= end) return;
  const int ntok = end - begin;
  const int ntiles = (ntok + T::TT - 1) / T::TT;
  const int n8 = d.nq[c];   // INT8-codes prefix (single-entry segments are read from their FP16 rows)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);   // provably warp-uniform
  const int lane = threadIdx.x & 31;
  const size_t cbase = (size_t)c * d.cap;
  const uint32_t sbase = smem_u32(smem);
  int* s_row = reinterpret_cast<int*>(smem + T::OFF_ROW);
  int* s_seg = reinterpret_cast<int*>(smem + T::OFF_SEG);
  const bool all8 = end <= n8;                               // INT8-only split: compact slots
  const int nstage = all8 ? T::STAGES8 : T::STAGES16;
  const uint32_t slotb = all8 ? T::SLOT8 : T::SLOT16;
  const uint32_t vofs = all8 ? T::SUB : T::NSUB * T::SUB;

  if (!rows_staged) {   // (an FP16 part's rows may have been staged beside the unit list)
    for (int j = threadIdx.x; j < ntok; j += kMmaWarps * 32) {
      const int sl = __ldg(d.slot + cbase + begin + j);
      const bool codes = begin + j < n8;
      s_row[j] = codes ? code_row(cbase, sl, d.Hkv, h) : (int)((cbase + sl) * d.Hkv + h);
      s_seg[j] = codes ? __ldg(d.seg + cbase + begin + j) : -1;
    }
  }
  __syncthreads();
  // one INT8 segment for the whole split (the bulk case): integer tensor-core (IMMA) path
  const bool bulk8 = __shfl_sync(0xffffffffu, (int)(all8 && s_seg[0] == s_seg[ntok - 1]), 0) != 0;
  if (lane == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(sbase + T::OFF_BAR + 8 * (warp * 8 + s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const uint32_t ring = sbase + warp * T::RING;
  const uint32_t bars = sbase + T::OFF_BAR + 8 * warp * 8;
  if constexpr (BULK) {
    if (bulk8) {
      attend_int8_split<D, G>(d, maps, c, c0, h, split, begin, end, ntok, ntiles, warp, lane, q, qscale, s_row,
                              s_seg[0], smem, sbase);
      return;
    }
  }
  for (int i = 0; i < nstage && warp + kMmaWarps * i < ntiles; ++i)
    issue_tile<D, G>(maps, s_row, warp + kMmaWarps * i, ntok, begin, n8, ring + i * slotb, vofs, bars + 8 * i);

  const int Hq = d.Hq;
  const int gq = lane >> 2, cq = lane & 3;            // MMA groupID / thread-in-group
  uint16_t* sPh = reinterpret_cast<uint16_t*>(smem + T::OFF_P) + warp * 2 * 8 * T::TT;
  uint16_t* sPl = sPh + 8 * T::TT;
  float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.sld;
  const int hA = 2 * cq, hB = 2 * cq + 1;
  const bool realA = hA < G, realB = hB < G;

  if (begin >= n8) {
    // ====== FP16-only split: ldmatrix fragments in natural order (conflict-free on the
    // swizzled ring), exact fp16 q / K, P hi+lo, O in natural dim order ======
    uint32_t bn[T::KSTEPS][2];
    {
      const __half* qn = q + ((size_t)(c - c0) * Hq + (size_t)h * G + gq) * D + 2 * cq;
#pragma unroll
      for (int kk = 0; kk < T::KSTEPS; ++kk) {
        bn[kk][0] = gq < G ? *reinterpret_cast<const uint32_t*>(qn + 16 * kk) : 0u;
        bn[kk][1] = gq < G ? *reinterpret_cast<const uint32_t*>(qn + 16 * kk + 8) : 0u;
      }
    }
    float mA = -INFINITY, mB = -INFINITY, zA = 0.f, zB = 0.f;
    float O[T::MT][4];
#pragma unroll
    for (int mt = 0; mt < T::MT; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) O[mt][i] = 0.f;
    const int lr = (lane & 7) + 8 * ((lane >> 3) & 1), lc = lane >> 4;   // q.K ldmatrix row / chunk
    const int vr = (lane & 7) + 8 * (lane >> 4), vc = (lane >> 3) & 1;   // P.V ldmatrix.trans row / chunk
    for (int it = 0; warp + kMmaWarps * it < ntiles; ++it) {
      const int k = warp + kMmaWarps * it;
      const int s = it % nstage;
      const uint32_t kb = ring + s * slotb;
      const uint32_t vb = kb + vofs;
      mbar_wait(bars + 8 * s, (it / nstage) & 1);
      const int tb = begin + k * T::TT;
      const int nvalid = __shfl_sync(0xffffffffu, min(T::TT, end - tb), 0);
      if (nvalid < T::TT) {
        // tail tile: rows beyond the split were never written; zero their V lines so
        // 0-probability rows cannot inject non-finite garbage into P.V
        for (int e = lane; e < (T::TT - nvalid) * T::NSUB * 8; e += 32) {
          const int r = nvalid + e / (T::NSUB * 8), rem = e % (T::NSUB * 8);
          asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(vb + (rem >> 3) * T::SUB + r * 128 + (rem & 7) * 16),
                       "r"(0u) : "memory");
        }
        __syncwarp();
      }
      float ca[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < T::KSTEPS; ++kk) {
        const int ch = 2 * kk + lc;
        uint32_t a[4];
        ldsm_x4(kb + (ch >> 3) * T::SUB + lr * 128 + (((ch & 7) ^ (lr & 7)) << 4), a);
        mma16816(ca[kk & 1], a, bn[kk][0], bn[kk][1]);
      }
      const int t0 = tb + gq, t1 = tb + gq + 8;
      const bool v0 = gq < nvalid, v1 = gq + 8 < nvalid;
      const float s0 = v0 ? (ca[0][0] + ca[1][0]) * qscale : -INFINITY;
      const float s1 = v0 ? (ca[0][1] + ca[1][1]) * qscale : -INFINITY;
      const float s2 = v1 ? (ca[0][2] + ca[1][2]) * qscale : -INFINITY;
      const float s3 = v1 ? (ca[0][3] + ca[1][3]) * qscale : -INFINITY;
      if (realA) {
        if (v0) scoreg[(size_t)hA * d.sld + t0] = s0;
        if (v1) scoreg[(size_t)hA * d.sld + t1] = s2;
      }
      if (realB) {
        if (v0) scoreg[(size_t)hB * d.sld + t0] = s1;
        if (v1) scoreg[(size_t)hB * d.sld + t1] = s3;
      }
      float tA = fmaxf(s0, s2), tB = fmaxf(s1, s3);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, o));
        tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, o));
      }
      const float nA = fmaxf(mA, tA), nB = fmaxf(mB, tB);
      const float cA = (mA == nA) ? 1.f : expf(mA - nA), cB = (mB == nB) ? 1.f : expf(mB - nB);
      const float p0 = (v0 && realA) ? expf(s0 - nA) : 0.f, p2 = (v1 && realA) ? expf(s2 - nA) : 0.f;
      const float p1 = (v0 && realB) ? expf(s1 - nB) : 0.f, p3 = (v1 && realB) ? expf(s3 - nB) : 0.f;
      zA = zA * cA + (p0 + p2);
      zB = zB * cB + (p1 + p3);
      mA = nA;
      mB = nB;
      {
        const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
        const __half h2 = __float2half_rn(p2), h3 = __float2half_rn(p3);
        sPh[hA * T::TT + gq] = __half_as_ushort(h0);
        sPh[hA * T::TT + gq + 8] = __half_as_ushort(h2);
        sPh[hB * T::TT + gq] = __half_as_ushort(h1);
        sPh[hB * T::TT + gq + 8] = __half_as_ushort(h3);
        sPl[hA * T::TT + gq] = __half_as_ushort(__float2half_rn(p0 - __half2float(h0)));
        sPl[hA * T::TT + gq + 8] = __half_as_ushort(__float2half_rn(p2 - __half2float(h2)));
        sPl[hB * T::TT + gq] = __half_as_ushort(__float2half_rn(p1 - __half2float(h1)));
        sPl[hB * T::TT + gq + 8] = __half_as_ushort(__float2half_rn(p3 - __half2float(h3)));
      }
      if (cA != 1.f || cB != 1.f) {
#pragma unroll
        for (int mt = 0; mt < T::MT; ++mt) {
          O[mt][0] *= cA; O[mt][1] *= cB; O[mt][2] *= cA; O[mt][3] *= cB;
        }
      }
      __syncwarp();
      const uint32_t ph0 = *reinterpret_cast<const uint32_t*>(sPh + gq * T::TT + 2 * cq);
      const uint32_t ph1 = *reinterpret_cast<const uint32_t*>(sPh + gq * T::TT + 2 * cq + 8);
      const uint32_t pl0 = *reinterpret_cast<const uint32_t*>(sPl + gq * T::TT + 2 * cq);
      const uint32_t pl1 = *reinterpret_cast<const uint32_t*>(sPl + gq * T::TT + 2 * cq + 8);
#pragma unroll
      for (int mt = 0; mt < T::MT; ++mt) {
        const int ch = 2 * mt + vc;
        uint32_t a[4];
        ldsm_x4_t(vb + (ch >> 3) * T::SUB + vr * 128 + (((ch & 7) ^ (vr & 7)) << 4), a);
        mma16816(O[mt], a, ph0, ph1);
        mma16816(O[mt], a, pl0, pl1);
      }
      __syncwarp();
      const int kn = k + kMmaWarps * nstage;
      if (kn < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_tile<D, G>(maps, s_row, kn, ntok, begin, n8, kb, vofs, bars + 8 * s);
      }
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      zA += __shfl_xor_sync(0xffffffffu, zA, o);
      zB += __shfl_xor_sync(0xffffffffu, zB, o);
    }
    __syncthreads();
    float* wacc = reinterpret_cast<float*>(smem);
    float* wm = wacc + kMmaWarps * G * D;
    float* wz = wm + kMmaWarps * G;
#pragma unroll
    for (int mt = 0; mt < T::MT; ++mt) {
      const int d0 = 16 * mt + gq;
      if (realA) {
        wacc[(warp * G + hA) * D + d0] = O[mt][0];
        wacc[(warp * G + hA) * D + d0 + 8] = O[mt][2];
      }
      if (realB) {
        wacc[(warp * G + hB) * D + d0] = O[mt][1];
        wacc[(warp * G + hB) * D + d0 + 8] = O[mt][3];
      }
    }
    if (gq == 0) {
      if (realA) { wm[warp * G + hA] = mA; wz[warp * G + hA] = zA; }
      if (realB) { wm[warp * G + hB] = mB; wz[warp * G + hB] = zB; }
    }
    __syncthreads();
    merge_warps<D, G>(d, c, h, split, wacc, wm, wz);
    return;
  }

  // exact q B-fragments (head gq, physical dims 16kk+4cq..+3); zero for padding heads
  uint32_t bq[T::KSTEPS][2];
  {
    const __half* qp = q + ((size_t)(c - c0) * Hq + (size_t)h * G + gq) * D + 4 * cq;
#pragma unroll
    for (int kk = 0; kk < T::KSTEPS; ++kk) {
      uint2 w = make_uint2(0u, 0u);
      if (gq < G) w = *reinterpret_cast<const uint2*>(qp + 16 * kk);
      bq[kk][0] = w.x;
      bq[kk][1] = w.y;
    }
  }
  uint32_t bh[T::KSTEPS][2], bl[T::KSTEPS][2];   // q * k_scale * 2^7, hi / lo
  int bseg = -1;
  float vsc[T::DS];                               // V scale of segment vseg, this thread's dim slice
  int vseg = -1;
  float mA = -INFINITY, mB = -INFINITY, zA = 0.f, zB = 0.f;
  float O[T::MT][4];
#pragma unroll
  for (int mt = 0; mt < T::MT; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) O[mt][i] = 0.f;
  const float* ksc_c = d.ksc + ((size_t)c * d.smax * d.Hkv + h) * D;
  const float* vsc_c = d.vsc + ((size_t)c * d.smax * d.Hkv + h) * D;
  const size_t seg_stride = (size_t)d.Hkv * D;

  for (int it = 0; warp + kMmaWarps * it < ntiles; ++it) {
    const int k = warp + kMmaWarps * it;
    const int s = it % nstage;
    const uint32_t kb = ring + s * slotb;
    const uint32_t vb = kb + vofs;
    mbar_wait(bars + 8 * s, (it / nstage) & 1);
    const int tb = begin + k * T::TT;                         // first entry of the tile
    const int tl = min(tb + T::TT, end) - 1;                  // last valid entry
    const bool tile16 = __shfl_sync(0xffffffffu, (int)(tb >= n8), 0) != 0;   // warp-uniform branches
    const bool tile8 = __shfl_sync(0xffffffffu, (int)(!tile16 && tl < n8 && s_seg[tb - begin] == s_seg[tl - begin]), 0) != 0;
    // four independent accumulator chains (k-step parity x hi/lo) keep the HMMA pipe busy
    float ca[4][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    float sfix = qscale;
    const int r0 = gq, r1 = gq + 8;
    // ================= q.K^T =================
    if (tile16) {
#pragma unroll
      for (int kk = 0; kk < T::KSTEPS; ++kk) {
        const uint32_t off = 8u * (cq & 1);
        const uint2 x0 = lds64(fp16_chunk<D>(kb, r0, 16 * kk + 8 * (cq >> 1)) + off);
        const uint2 x1 = lds64(fp16_chunk<D>(kb, r1, 16 * kk + 8 * (cq >> 1)) + off);
        const uint32_t a[4] = {x0.x, x1.x, x0.y, x1.y};
        mma16816(ca[kk & 3], a, bq[kk][0], bq[kk][1]);
      }
    } else if (tile8) {
      const int sg = s_seg[tb - begin];
      if (sg != bseg) {
        const float* ks = ksc_c + (size_t)sg * seg_stride + 4 * cq;
#pragma unroll
        for (int kk = 0; kk < T::KSTEPS; ++kk) {
          const float4 k4 = __ldg(reinterpret_cast<const float4*>(ks + 16 * kk));
          const float2 q01 = __half22float2(*reinterpret_cast<const __half2*>(&bq[kk][0]));
          const float2 q23 = __half22float2(*reinterpret_cast<const __half2*>(&bq[kk][1]));
          split_h2(q01.x * (k4.x * 128.f), q01.y * (k4.y * 128.f), bh[kk][0], bl[kk][0]);
          split_h2(q23.x * (k4.z * 128.f), q23.y * (k4.w * 128.f), bh[kk][1], bl[kk][1]);
        }
        bseg = sg;
      }
#pragma unroll
      for (int kk = 0; kk < T::KSTEPS; ++kk) {
        const uint32_t w0 = lds32(int8_chunk(kb, r0, 16 * kk + 4 * cq));
        const uint32_t w1 = lds32(int8_chunk(kb, r1, 16 * kk + 4 * cq));
        uint32_t a[4];
        codes4_to_h2(w0, a[0], a[2]);
        codes4_to_h2(w1, a[1], a[3]);
        mma16816(ca[2 * (kk & 1)], a, bh[kk][0], bh[kk][1]);
        mma16816(ca[2 * (kk & 1) + 1], a, bl[kk][0], bl[kk][1]);
      }
      sfix = qscale * (1.f / 128.f);
    } else {
      const int t0 = tb + gq, t1 = tb + gq + 8;
      const bool q0 = t0 < n8 && t0 < end, q1 = t1 < n8 && t1 < end;
      const float* ks0 = q0 ? ksc_c + (size_t)s_seg[t0 - begin] * seg_stride + 4 * cq : nullptr;
      const float* ks1 = q1 ? ksc_c + (size_t)s_seg[t1 - begin] * seg_stride + 4 * cq : nullptr;
#pragma unroll
      for (int kk = 0; kk < T::KSTEPS; ++kk) {
        uint32_t ah[4], al[4];
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
          const int row = rr ? r1 : r0;
          if (rr ? q1 : q0) {
            const float4 k4 = __ldg(reinterpret_cast<const float4*>((rr ? ks1 : ks0) + 16 * kk));
            float2 f[4];
            code8_to_f2(make_uint2(lds32(int8_chunk(kb, row, 16 * kk + 4 * cq)), 0u), f);
            split_h2(f[0].x * k4.x, f[0].y * k4.y, ah[rr], al[rr]);
            split_h2(f[1].x * k4.z, f[1].y * k4.w, ah[rr + 2], al[rr + 2]);
          } else {
            const uint2 x = lds64(fp16_chunk<D>(kb, row, 16 * kk + 8 * (cq >> 1)) + 8u * (cq & 1));
            ah[rr] = x.x; ah[rr + 2] = x.y; al[rr] = 0u; al[rr + 2] = 0u;
          }
        }
        mma16816(ca[2 * (kk & 1)], ah, bq[kk][0], bq[kk][1]);
        mma16816(ca[2 * (kk & 1) + 1], al, bq[kk][0], bq[kk][1]);
      }
    }
    float cacc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) cacc[i] = (ca[0][i] + ca[2][i]) + (ca[1][i] + ca[3][i]);
    // ================= online softmax on the fragments =================
    float cA, cB;
    {
      const int t0 = tb + gq, t1 = tb + gq + 8;
      const bool v0 = t0 < end, v1 = t1 < end;
      const float s0 = v0 ? cacc[0] * sfix : -INFINITY, s1 = v0 ? cacc[1] * sfix : -INFINITY;
      const float s2 = v1 ? cacc[2] * sfix : -INFINITY, s3 = v1 ? cacc[3] * sfix : -INFINITY;
      if (realA) {
        if (v0) scoreg[(size_t)hA * d.sld + t0] = s0;
        if (v1) scoreg[(size_t)hA * d.sld + t1] = s2;
      }
      if (realB) {
        if (v0) scoreg[(size_t)hB * d.sld + t0] = s1;
        if (v1) scoreg[(size_t)hB * d.sld + t1] = s3;
      }
      float tA = fmaxf(s0, s2), tB = fmaxf(s1, s3);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, o));
        tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, o));
      }
      const float nA = fmaxf(mA, tA), nB = fmaxf(mB, tB);
      cA = (mA == nA) ? 1.f : expf(mA - nA);
      cB = (mB == nB) ? 1.f : expf(mB - nB);
      const float p0 = (v0 && realA) ? expf(s0 - nA) : 0.f, p2 = (v1 && realA) ? expf(s2 - nA) : 0.f;
      const float p1 = (v0 && realB) ? expf(s1 - nB) : 0.f, p3 = (v1 && realB) ? expf(s3 - nB) : 0.f;
      zA = zA * cA + (p0 + p2);
      zB = zB * cB + (p1 + p3);
      mA = nA;
      mB = nB;
      // P (hi, lo) as fp16 [head][entry], entry order permuted for the P.V B fragment:
      // row r -> column (r&3)*4... stored by physical entry; reader takes entries 4c..4c+3
      const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
      const __half h2 = __float2half_rn(p2), h3 = __float2half_rn(p3);
      sPh[hA * T::TT + r0] = __half_as_ushort(h0);
      sPh[hA * T::TT + r1] = __half_as_ushort(h2);
      sPh[hB * T::TT + r0] = __half_as_ushort(h1);
      sPh[hB * T::TT + r1] = __half_as_ushort(h3);
      sPl[hA * T::TT + r0] = __half_as_ushort(__float2half_rn(p0 - __half2float(h0)));
      sPl[hA * T::TT + r1] = __half_as_ushort(__float2half_rn(p2 - __half2float(h2)));
      sPl[hB * T::TT + r0] = __half_as_ushort(__float2half_rn(p1 - __half2float(h1)));
      sPl[hB * T::TT + r1] = __half_as_ushort(__float2half_rn(p3 - __half2float(h3)));
    }
    if (cA != 1.f || cB != 1.f) {
#pragma unroll
      for (int mt = 0; mt < T::MT; ++mt) {
        O[mt][0] *= cA; O[mt][1] *= cB; O[mt][2] *= cA; O[mt][3] *= cB;
      }
    }
    __syncwarp();
    // B fragments: head gq, entries 4cq..4cq+3 (k-indices 2c,2c+1 | 2c+8,2c+9)
    const uint2 pbh = *reinterpret_cast<const uint2*>(sPh + gq * T::TT + 4 * cq);
    const uint2 pbl = *reinterpret_cast<const uint2*>(sPl + gq * T::TT + 4 * cq);
    // ================= P.V =================
    const int e0 = 4 * cq;                              // this thread's 4 entries (stage rows)
    if (tile16) {
      // FP16 rows e0..e0+3, dims [DS*gq, +DS): 16-byte chunks, paired across rows by PRMT
#pragma unroll
      for (int half = 0; half < T::DS / 8; ++half) {
        uint4 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          x[j] = lds128(fp16_chunk<D>(vb, e0 + j, T::DS * gq + 8 * half));
          // rows past the split's end were never loaded (stale shared memory, possibly NaN bit
          // patterns): P is 0 there, but 0 * NaN is not, so zero them
          if (tb + e0 + j >= end) x[j] = make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int m4 = 0; m4 < 4; ++m4) {
          const int mt = half * 4 + m4;
          const uint32_t w0 = (&x[0].x)[m4], w1 = (&x[1].x)[m4], w2 = (&x[2].x)[m4], w3 = (&x[3].x)[m4];
          const uint32_t a[4] = {__byte_perm(w0, w1, 0x5410), __byte_perm(w0, w1, 0x7632),
                                 __byte_perm(w2, w3, 0x5410), __byte_perm(w2, w3, 0x7632)};
          mma16816(O[mt], a, pbh.x, pbh.y);
          mma16816(O[mt], a, pbl.x, pbl.y);
        }
      }
    } else if (tile8) {
      const int sg = s_seg[tb - begin];
      if (sg != vseg) {
        const float* vs = vsc_c + (size_t)sg * seg_stride + T::DS * gq;
#pragma unroll
        for (int i = 0; i < T::DS; i += 4) {
          const float4 v4 = __ldg(reinterpret_cast<const float4*>(vs + i));
          vsc[i] = v4.x; vsc[i + 1] = v4.y; vsc[i + 2] = v4.z; vsc[i + 3] = v4.w;
        }
        vseg = sg;
      }
      uint32_t wv[4][T::DS / 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if constexpr (T::DS == 16) {
          const uint4 x = lds128(int8_chunk(vb, e0 + j, T::DS * gq));
          wv[j][0] = x.x ^ 0x80808080u; wv[j][1] = x.y ^ 0x80808080u;
          wv[j][2] = x.z ^ 0x80808080u; wv[j][3] = x.w ^ 0x80808080u;
        } else {
          const uint2 x = lds64(int8_chunk(vb, e0 + j, T::DS * gq));
          wv[j][0] = x.x ^ 0x80808080u; wv[j][1] = x.y ^ 0x80808080u;
        }
      }
#pragma unroll
      for (int mt = 0; mt < T::MT; ++mt) {
        const int wd = mt >> 1, bt = 2 * (mt & 1);
        const uint32_t sel0 = (uint32_t)((4 + bt) << 8 | bt), sel1 = sel0 + 0x101u;
        const uint32_t a[4] = {pair_codes(wv[0][wd], wv[1][wd], sel0), pair_codes(wv[0][wd], wv[1][wd], sel1),
                               pair_codes(wv[2][wd], wv[3][wd], sel0), pair_codes(wv[2][wd], wv[3][wd], sel1)};
        float t4[4] = {0.f, 0.f, 0.f, 0.f};
        mma16816(t4, a, pbh.x, pbh.y);
        mma16816(t4, a, pbl.x, pbl.y);
        const float sa = vsc[2 * mt], sb = vsc[2 * mt + 1];
        O[mt][0] = fmaf(t4[0], sa, O[mt][0]); O[mt][1] = fmaf(t4[1], sa, O[mt][1]);
        O[mt][2] = fmaf(t4[2], sb, O[mt][2]); O[mt][3] = fmaf(t4[3], sb, O[mt][3]);
      }
    } else {
      // mixed: per row, fp32 values (FP16 as is, INT8 code * scale), split hi/lo; 8 dims at a time
#pragma unroll
      for (int half = 0; half < T::DS / 8; ++half) {
        uint32_t vh[4][4], vl[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int tok = tb + e0 + j;
          const int i = 8 * half;
          if (tok < end && tok < n8) {
            const float* vs = vsc_c + (size_t)s_seg[tok - begin] * seg_stride + T::DS * gq + i;
            float2 f[4];
            code8_to_f2(lds64(int8_chunk(vb, e0 + j, T::DS * gq + i)), f);
            const float4 s0 = __ldg(reinterpret_cast<const float4*>(vs));
            const float4 s1 = __ldg(reinterpret_cast<const float4*>(vs + 4));
            split_h2(f[0].x * s0.x, f[0].y * s0.y, vh[j][0], vl[j][0]);
            split_h2(f[1].x * s0.z, f[1].y * s0.w, vh[j][1], vl[j][1]);
            split_h2(f[2].x * s1.x, f[2].y * s1.y, vh[j][2], vl[j][2]);
            split_h2(f[3].x * s1.z, f[3].y * s1.w, vh[j][3], vl[j][3]);
          } else if (tok < end) {
            const uint4 x = lds128(fp16_chunk<D>(vb, e0 + j, T::DS * gq + i));
            vh[j][0] = x.x; vh[j][1] = x.y; vh[j][2] = x.z; vh[j][3] = x.w;
            vl[j][0] = vl[j][1] = vl[j][2] = vl[j][3] = 0u;
          } else {
            vh[j][0] = vh[j][1] = vh[j][2] = vh[j][3] = 0u;
            vl[j][0] = vl[j][1] = vl[j][2] = vl[j][3] = 0u;
          }
        }
#pragma unroll
        for (int m4 = 0; m4 < 4; ++m4) {
          const int mt = half * 4 + m4;
          const uint32_t ah[4] = {__byte_perm(vh[0][m4], vh[1][m4], 0x5410), __byte_perm(vh[0][m4], vh[1][m4], 0x7632),
                                  __byte_perm(vh[2][m4], vh[3][m4], 0x5410), __byte_perm(vh[2][m4], vh[3][m4], 0x7632)};
          const uint32_t al[4] = {__byte_perm(vl[0][m4], vl[1][m4], 0x5410), __byte_perm(vl[0][m4], vl[1][m4], 0x7632),
                                  __byte_perm(vl[2][m4], vl[3][m4], 0x5410), __byte_perm(vl[2][m4], vl[3][m4], 0x7632)};
          mma16816(O[mt], ah, pbh.x, pbh.y);
          mma16816(O[mt], ah, pbl.x, pbl.y);
          mma16816(O[mt], al, pbh.x, pbh.y);
        }
      }
    }
    __syncwarp();   // slot and sP are reused after this
    const int kn = k + kMmaWarps * nstage;
    if (kn < ntiles) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_tile<D, G>(maps, s_row, kn, ntok, begin, n8, kb, vofs, bars + 8 * s);
    }
  }

  // ---- epilogue: per-warp (m, z, O) -> smem -> split partials ------------------------------
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    zA += __shfl_xor_sync(0xffffffffu, zA, o);
    zB += __shfl_xor_sync(0xffffffffu, zB, o);
  }
  __syncthreads();   // every warp has drained its ring: it may be reused as scratch
  float* wacc = reinterpret_cast<float*>(smem);
  float* wm = wacc + kMmaWarps * G * D;
  float* wz = wm + kMmaWarps * G;
#pragma unroll
  for (int mt = 0; mt < T::MT; ++mt) {
    const int d0 = T::DS * gq + 2 * mt;
    if (realA) {
      wacc[(warp * G + hA) * D + d0] = O[mt][0];
      wacc[(warp * G + hA) * D + d0 + 1] = O[mt][2];
    }
    if (realB) {
      wacc[(warp * G + hB) * D + d0] = O[mt][1];
      wacc[(warp * G + hB) * D + d0 + 1] = O[mt][3];
    }
  }
  if (gq == 0) {
    if (realA) { wm[warp * G + hA] = mA; wz[warp * G + hA] = zA; }
    if (realB) { wm[warp * G + hB] = mB; wz[warp * G + hB] = zB; }
  }
  __syncthreads();
  merge_warps<D, G>(d, c, h, split, wacc, wm, wz);
}

// ============================================================================================
// FP16-part streaming kernel (D = 64 / 128): every partial slot whose entries are all read as
// FP16 rows (the FP16 window beside a bulk INT8 segment, single-entry INT8 segments, FP16-only
// caches) is a unit (cache, KV head, part), and one consumer warp computes a whole unit, so a
// unit needs no cross-warp merge or barrier. A persistent grid: per CTA one producer warp keeps
// each of the 4 consumer warps' private rings of 16-entry K/V tiles full, round-robin and
// without blocking (a warp whose ring is full is skipped), and hands a warp its next unit as
// soon as the previous unit's tiles are issued -- the next unit's slot indices are already in
// registers -- so HBM keeps streaming across unit boundaries instead of paying a short CTA's
// ramp (slot lookups, first TMA round trip, merge) per unit.
//   warp 4     producer: unit descriptors (32 candidates per ballot, static stride over the
//              grid), row coordinates, 128B-swizzled gather4 of each tile's K and V rows. A tile
//              past the unit's end repeats the unit's last row (constant tx bytes; its
//              probabilities are 0 and the repeated V rows are finite).
//   warps 0-3  consumers: per tile q.K^T and P.V on mma.sync with the general kernel's FP16
//              arithmetic (exact fp16 q / K, P split hi + lo), scores to the EMA scratch, online
//              softmax; at the unit's end the warp writes the unit's partial slot directly.
template <int D, int G>
struct TsP {
  static constexpr int TT = 16;
  static constexpr int NSUB = D / 64;
  static constexpr int SUB = TT * 128;
  static constexpr int SLOT = 2 * NSUB * SUB;                        // K + V tile
  static constexpr int UMAX = kSplitTokens + kAbsorbTokens;          // entries per unit (max)
  static constexpr int ROWS = (UMAX + TT - 1) / TT * TT;
  static constexpr int W = kMmaWarps;
  static constexpr int FIXED = W * ROWS * 4 + W * 2 * 8 * TT * 2 + W * 2 * 16 + 1024;
  static constexpr int BUDGET = (D == 128 ? 111 : 72) * 1024;        // 2 (D=128) / 3 (D=64) CTAs per SM
  static constexpr int NSW0 = (BUDGET - FIXED) / (W * SLOT);
  static constexpr int NSW = NSW0 > 8 ? 8 : NSW0;                   // ring slots per consumer warp
  static constexpr int OFF_ROW = W * NSW * SLOT;
  static constexpr int OFF_P = OFF_ROW + W * ROWS * 4;
  static constexpr int OFF_UNIT = OFF_P + W * 2 * 8 * TT * 2;       // [W][2] int4
  static constexpr int OFF_BAR = OFF_UNIT + W * 2 * 16;
  // barriers: full / empty per ring slot, full / empty per unit descriptor
  static constexpr int B_FULL = 0, B_EMPTY = W * NSW, B_UFULL = 2 * W * NSW, B_UEMPTY = 2 * W * NSW + 2 * W,
                       N_BAR = 2 * W * NSW + 4 * W;
  static constexpr int SMEM = OFF_BAR + 8 * N_BAR;
  static constexpr int THREADS = (W + 1) * 32;
  static constexpr int KSTEPS = D / 16, MT = D / 16;
  static_assert(NSW >= 3, "ring depth per warp");
  static_assert(SMEM <= BUDGET, "CTAs per SM");
};

// A unit: the FP16 side of a split in cut mode (odd slot), or a whole split whose entries are
// all read as FP16 otherwise (kind 1); with d.scodes (D = 128, no tcgen05 grid) also the codes
// side of a split when it lies in one lossy segment (kind 0; sg = that segment).
__device__ __forceinline__ bool stream_unit(const Dev& d, int c, int sp, int kind, int& p, int& b, int& e, int& sg) {
  const int n = d.len[c], nq = d.nq[c];
  sg = -1;
  if (kind) {
    p = d.cut_nq ? 2 * sp + 1 : 2 * sp;
    part_range(d, sp, p & 1, n, nq, b, e);
    return b < e && b >= nq;
  }
  p = 2 * sp;
  part_range(d, sp, 0, n, nq, b, e);
  if (b >= e) return false;
  sg = __ldg(d.seg + (size_t)c * d.cap + b);
  return sg == __ldg(d.seg + (size_t)c * d.cap + e - 1);
}

__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}

// Called by every thread of the CTA (warps past the producer idle); returns with every
// barrier of its smem carve-up invalidated, so the caller may reuse the shared memory.
template <int D, int G>
__device__ __forceinline__ void fp16_units(const Dev& d, const Maps& maps, int c0, int ccount,
                                           const __half* __restrict__ q, float qscale, uint8_t* smem) {
  using T = TsP<D, G>;
  constexpr int NSW = T::NSW, TT = T::TT, W = T::W;
  const uint32_t sbase = smem_u32(smem);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  const int lane = threadIdx.x & 31;
  const uint32_t bars = sbase + T::OFF_BAR;
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  int4* s_unit = reinterpret_cast<int4*>(smem + T::OFF_UNIT);
  if (threadIdx.x == 0) {
    for (int i = 0; i < T::N_BAR; ++i) mbar_init(bar(i), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int Hkv = d.Hkv, nsp = d.live_splits;
  const bool codes = D == 128 && d.scodes;             // codes units on this kernel too
  const int kinds = codes ? 2 : 1;
  const int total = ccount * Hkv * nsp * kinds;

  if (warp == W) {
    // ===================================== producer =====================================
    // Candidates in (split, kind)-major order, (cache, KV head) fastest, strided statically over
    // the grid: every CTA then gets every kind of unit from every layer (units differ in length:
    // pyramid budgets, empty second splits, codes vs FP16). A (cache, head, split, kind) order
    // gave each CTA one fixed (split, kind) residue whenever the grid size shared a factor with
    // the candidate period (Qwen pyramid: ends 16 -> 373 us); claiming candidates dynamically
    // put an atomic round trip on the producer's issue path (INT8 4K: +25 us).
    int base = (int)blockIdx.x - 32 * (int)gridDim.x;
    unsigned m = 0;
    int c = 0, h = 0, p = 0, b = 0, e = 0, sg = -1;  // this lane's candidate
    const int pairs = ccount * Hkv;
    auto next = [&](int& ic, int& ih, int& ip, int& ib, int& ie, int& isg) -> bool {
      while (!m) {
        base += 32 * (int)gridDim.x;
        if (base >= total) return false;
        const int k = base + lane * (int)gridDim.x;
        bool ok = false;
        if (k < total) {
          const int sk = k / pairs, pr = k - sk * pairs;   // (split, kind), (cache, head)
          const int kind = codes ? (sk & 1) : 1, sp = codes ? (sk >> 1) : sk;
          h = pr % Hkv;
          c = c0 + pr / Hkv;
          ok = stream_unit(d, c, sp, kind, p, b, e, sg);
        }
        m = __ballot_sync(0xffffffffu, ok);
      }
      const int L = __ffs(m) - 1;
      m &= m - 1;
      ic = __shfl_sync(0xffffffffu, c, L); ih = __shfl_sync(0xffffffffu, h, L);
      ip = __shfl_sync(0xffffffffu, p, L); ib = __shfl_sync(0xffffffffu, b, L);
      ie = __shfl_sync(0xffffffffu, e, L); isg = __shfl_sync(0xffffffffu, sg, L);
      return true;
    };
    constexpr int SPL = T::ROWS / 32;
    // the next unit, slot indices already loaded (rows past its end repeat the last entry)
    int nc = 0, nh = 0, np = 0, nb = 0, ne = 0, nsg = -1;
    int nv[SPL];
    auto prefetch = [&]() -> bool {
      if (!next(nc, nh, np, nb, ne, nsg)) return false;
      const int* sl = d.slot + (size_t)nc * d.cap + nb;
      const int nt = ne - nb;
#pragma unroll
      for (int i = 0; i < SPL; ++i) nv[i] = __ldg(sl + min(lane + 32 * i, nt - 1));
      return true;
    };
    bool have = prefetch();
    int tcur[W], tnum[W], gw[W], uc[W];
    bool ended[W], ucode[W];
#pragma unroll
    for (int w = 0; w < W; ++w) { tcur[w] = 0; tnum[w] = 0; gw[w] = 0; uc[w] = 0; ended[w] = false; ucode[w] = false; }
    int live = W;
    while (live) {
#pragma unroll
      for (int w = 0; w < W; ++w) {
        if (ended[w]) continue;
        int* rows = reinterpret_cast<int*>(smem + T::OFF_ROW) + w * T::ROWS;
        if (tcur[w] == tnum[w]) {
          // warp w's unit is fully issued: hand it the next one (or its end marker)
          const int k = uc[w] & 1;
          if (uc[w] >= 2 && !mbar_test(bar(T::B_UEMPTY + 2 * w + k), ((uc[w] >> 1) - 1) & 1)) continue;
          if (!have) {
            if (lane == 0) {
              s_unit[2 * w + k] = make_int4(-1, 0, 0, 0);
              mbar_arrive(bar(T::B_UFULL + 2 * w + k));
            }
            ended[w] = true;
            --live;
            continue;
          }
          const size_t cb = (size_t)nc * d.cap;
          if (nsg >= 0) {                                 // code slots -> code rows
#pragma unroll
            for (int i = 0; i < SPL; ++i) rows[lane + 32 * i] = code_row(cb, nv[i], Hkv, nh);
          } else {
#pragma unroll
            for (int i = 0; i < SPL; ++i) rows[lane + 32 * i] = (int)((cb + nv[i]) * Hkv + nh);
          }
          const int ntok = ne - nb;
          __syncwarp();
          if (lane == 0) {
            s_unit[2 * w + k] = make_int4(nc, nh | (np << 8), nb | (ntok << 20), nsg);
            mbar_arrive(bar(T::B_UFULL + 2 * w + k));
          }
          ucode[w] = nsg >= 0;
          ++uc[w];
          tcur[w] = 0;
          tnum[w] = (ntok + TT - 1) / TT;
          have = prefetch();
        }
        // one tile for warp w if its next ring slot is free
        const int s = gw[w] % NSW, use = gw[w] / NSW;
        if (use > 0 && !mbar_test(bar(T::B_EMPTY + w * NSW + s), (use - 1) & 1)) continue;
        const uint32_t kb = sbase + (uint32_t)((w * NSW + s) * T::SLOT), vb = kb + T::NSUB * T::SUB;
        const uint32_t fb = bar(T::B_FULL + w * NSW + s);
        const bool leader = elect_one();
        const int t = tcur[w];
        if (ucode[w]) {   // 16 code rows of K and of V, one 128-byte line each
          if (leader) mbar_arrive_tx(fb, 2 * TT * 128);
#pragma unroll
          for (int g0 = 0; g0 < TT; g0 += 4) {
            const int4 r = *reinterpret_cast<const int4*>(rows + t * TT + g0);
            if (leader) {
              tma_gather4(kb + g0 * 128, &maps.kq_sw, r.x, r.y, r.z, r.w, fb, 0);
              tma_gather4(vb + g0 * 128, &maps.vq_sw, r.x, r.y, r.z, r.w, fb, 0);
            }
          }
        } else {
          if (leader) mbar_arrive_tx(fb, T::SLOT);
#pragma unroll
          for (int g0 = 0; g0 < TT; g0 += 4) {
            const int4 r = *reinterpret_cast<const int4*>(rows + t * TT + g0);
            if (leader) {
#pragma unroll
              for (int sub = 0; sub < T::NSUB; ++sub) {
                tma_gather4(kb + sub * T::SUB + g0 * 128, &maps.kf_sw, r.x, r.y, r.z, r.w, fb, sub * 64);
                tma_gather4(vb + sub * T::SUB + g0 * 128, &maps.vf_sw, r.x, r.y, r.z, r.w, fb, sub * 64);
              }
            }
          }
        }
        __syncwarp();
        ++tcur[w];
        ++gw[w];
      }
    }
  } else if (warp < W) {
    // ===================================== consumers =====================================
    const int Hq = d.Hq, npt = d.npart;
    const int gq = lane >> 2, cq = lane & 3;
    const int hA = 2 * cq, hB = 2 * cq + 1;
    const bool realA = hA < G, realB = hB < G;
    uint16_t* sPh = reinterpret_cast<uint16_t*>(smem + T::OFF_P) + warp * 2 * 8 * TT;
    uint16_t* sPl = sPh + 8 * TT;
    const int lr = (lane & 7) + 8 * ((lane >> 3) & 1), lc = lane >> 4;   // q.K ldmatrix row / chunk
    const int vr = (lane & 7) + 8 * (lane >> 4), vc = (lane >> 3) & 1;   // P.V ldmatrix.trans row / chunk
    int gtile = 0;                                                      // tiles consumed (ring position)
    for (int j = 0;; ++j) {
      const int k = j & 1;
      mbar_wait(bar(T::B_UFULL + 2 * warp + k), (j >> 1) & 1);
      const uint4 du = lds128(smem_u32(s_unit + 2 * warp + k));
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(T::B_UEMPTY + 2 * warp + k));
      const int c = (int)du.x;
      if (c < 0) break;
      const int h = (int)(du.y & 255u), part = (int)(du.y >> 8);
      const int begin = (int)(du.z & ((1u << 20) - 1u)), ntok = (int)(du.z >> 20);
      const int ntiles = (ntok + TT - 1) / TT;
      if constexpr (D == 128) {
        const int sg = (int)du.w;
        if (sg >= 0) {
          // ---- codes unit: one lossy segment, the general kernel's integer-tile arithmetic:
          // q.K^T on exact codes with q * k_scale * 2^7 split into fp16 hi + lo, P hi + lo on the
          // codes of V, the segment's V scale per output dim; head dims permuted (k-indices
          // {2c, 2c+1, 2c+8, 2c+9} of k-step kk = dims 16kk + 4c .. +3; output dims DS*g + 2mt + half)
          constexpr int DS = D / 8;
          const size_t srow = (((size_t)c * d.smax + sg) * Hkv + h) * D;
          uint32_t bh[T::KSTEPS][2], bl[T::KSTEPS][2];
          {
            const __half* qp = q + ((size_t)(c - c0) * Hq + (size_t)h * G + gq) * D + 4 * cq;
            const float* ks = d.ksc + srow + 4 * cq;
#pragma unroll
            for (int kk = 0; kk < T::KSTEPS; ++kk) {
              uint2 w = make_uint2(0u, 0u);
              if (gq < G) w = *reinterpret_cast<const uint2*>(qp + 16 * kk);
              const float4 k4 = __ldg(reinterpret_cast<const float4*>(ks + 16 * kk));
              const float2 q01 = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
              const float2 q23 = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
              split_h2(q01.x * (k4.x * 128.f), q01.y * (k4.y * 128.f), bh[kk][0], bl[kk][0]);
              split_h2(q23.x * (k4.z * 128.f), q23.y * (k4.w * 128.f), bh[kk][1], bl[kk][1]);
            }
          }
          float vsc[DS];
          {
            const float* vs = d.vsc + srow + DS * gq;
#pragma unroll
            for (int i = 0; i < DS; i += 4) {
              const float4 v4 = __ldg(reinterpret_cast<const float4*>(vs + i));
              vsc[i] = v4.x; vsc[i + 1] = v4.y; vsc[i + 2] = v4.z; vsc[i + 3] = v4.w;
            }
          }
          const float sfix = qscale * (1.f / 128.f);
          float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.sld;
          float mA = -INFINITY, mB = -INFINITY, zA = 0.f, zB = 0.f;
          float O[T::MT][4];
#pragma unroll
          for (int mt = 0; mt < T::MT; ++mt)
#pragma unroll
            for (int i = 0; i < 4; ++i) O[mt][i] = 0.f;
          for (int t = 0; t < ntiles; ++t, ++gtile) {
            const int s = gtile % NSW;
            const uint32_t kb = sbase + (uint32_t)((warp * NSW + s) * T::SLOT), vb = kb + T::NSUB * T::SUB;
            mbar_wait(bar(T::B_FULL + warp * NSW + s), (gtile / NSW) & 1);
            const int tb = begin + t * TT;
            const int nvalid = min(TT, begin + ntok - tb);
            float ca[4][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int kk = 0; kk < T::KSTEPS; ++kk) {
              const uint32_t w0 = lds32(int8_chunk(kb, gq, 16 * kk + 4 * cq));
              const uint32_t w1 = lds32(int8_chunk(kb, gq + 8, 16 * kk + 4 * cq));
              uint32_t a[4];
              codes4_to_h2(w0, a[0], a[2]);
              codes4_to_h2(w1, a[1], a[3]);
              mma16816(ca[2 * (kk & 1)], a, bh[kk][0], bh[kk][1]);
              mma16816(ca[2 * (kk & 1) + 1], a, bl[kk][0], bl[kk][1]);
            }
            float cacc[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) cacc[i] = (ca[0][i] + ca[2][i]) + (ca[1][i] + ca[3][i]);
            const int t0 = tb + gq, t1 = tb + gq + 8;
            const bool v0 = gq < nvalid, v1 = gq + 8 < nvalid;
            const float s0 = v0 ? cacc[0] * sfix : -INFINITY, s1 = v0 ? cacc[1] * sfix : -INFINITY;
            const float s2 = v1 ? cacc[2] * sfix : -INFINITY, s3 = v1 ? cacc[3] * sfix : -INFINITY;
            if (realA) {
              if (v0) scoreg[(size_t)hA * d.sld + t0] = s0;
              if (v1) scoreg[(size_t)hA * d.sld + t1] = s2;
            }
            if (realB) {
              if (v0) scoreg[(size_t)hB * d.sld + t0] = s1;
              if (v1) scoreg[(size_t)hB * d.sld + t1] = s3;
            }
            float tA = fmaxf(s0, s2), tB = fmaxf(s1, s3);
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
              tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, o));
              tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, o));
            }
            const float nA = fmaxf(mA, tA), nB = fmaxf(mB, tB);
            const float cA = (mA == nA) ? 1.f : expf(mA - nA), cB = (mB == nB) ? 1.f : expf(mB - nB);
            const float p0 = (v0 && realA) ? expf(s0 - nA) : 0.f, p2 = (v1 && realA) ? expf(s2 - nA) : 0.f;
            const float p1 = (v0 && realB) ? expf(s1 - nB) : 0.f, p3 = (v1 && realB) ? expf(s3 - nB) : 0.f;
            zA = zA * cA + (p0 + p2);
            zB = zB * cB + (p1 + p3);
            mA = nA;
            mB = nB;
            {
              const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
              const __half h2 = __float2half_rn(p2), h3 = __float2half_rn(p3);
              sPh[hA * TT + gq] = __half_as_ushort(h0);
              sPh[hA * TT + gq + 8] = __half_as_ushort(h2);
              sPh[hB * TT + gq] = __half_as_ushort(h1);
              sPh[hB * TT + gq + 8] = __half_as_ushort(h3);
              sPl[hA * TT + gq] = __half_as_ushort(__float2half_rn(p0 - __half2float(h0)));
              sPl[hA * TT + gq + 8] = __half_as_ushort(__float2half_rn(p2 - __half2float(h2)));
              sPl[hB * TT + gq] = __half_as_ushort(__float2half_rn(p1 - __half2float(h1)));
              sPl[hB * TT + gq + 8] = __half_as_ushort(__float2half_rn(p3 - __half2float(h3)));
            }
            if (cA != 1.f || cB != 1.f) {
#pragma unroll
              for (int mt = 0; mt < T::MT; ++mt) {
                O[mt][0] *= cA; O[mt][1] *= cB; O[mt][2] *= cA; O[mt][3] *= cB;
              }
            }
            __syncwarp();
            // B fragments: head gq, entries 4cq .. 4cq+3
            const uint2 pbh = *reinterpret_cast<const uint2*>(sPh + gq * TT + 4 * cq);
            const uint2 pbl = *reinterpret_cast<const uint2*>(sPl + gq * TT + 4 * cq);
            const int e0 = 4 * cq;
            uint32_t wv[4][DS / 4];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const uint4 x = lds128(int8_chunk(vb, e0 + jj, DS * gq));
              wv[jj][0] = x.x ^ 0x80808080u; wv[jj][1] = x.y ^ 0x80808080u;
              wv[jj][2] = x.z ^ 0x80808080u; wv[jj][3] = x.w ^ 0x80808080u;
            }
#pragma unroll
            for (int mt = 0; mt < T::MT; ++mt) {
              const int wd = mt >> 1, bt = 2 * (mt & 1);
              const uint32_t sel0 = (uint32_t)((4 + bt) << 8 | bt), sel1 = sel0 + 0x101u;
              const uint32_t a[4] = {pair_codes(wv[0][wd], wv[1][wd], sel0), pair_codes(wv[0][wd], wv[1][wd], sel1),
                                     pair_codes(wv[2][wd], wv[3][wd], sel0), pair_codes(wv[2][wd], wv[3][wd], sel1)};
              float t4[4] = {0.f, 0.f, 0.f, 0.f};
              mma16816(t4, a, pbh.x, pbh.y);
              mma16816(t4, a, pbl.x, pbl.y);
              const float sa = vsc[2 * mt], sb = vsc[2 * mt + 1];
              O[mt][0] = fmaf(t4[0], sa, O[mt][0]); O[mt][1] = fmaf(t4[1], sa, O[mt][1]);
              O[mt][2] = fmaf(t4[2], sb, O[mt][2]); O[mt][3] = fmaf(t4[3], sb, O[mt][3]);
            }
            __syncwarp();                               // slot and sP reads done
            if (lane == 0) mbar_arrive(bar(T::B_EMPTY + warp * NSW + s));
          }
#pragma unroll
          for (int o = 4; o < 32; o <<= 1) {
            zA += __shfl_xor_sync(0xffffffffu, zA, o);
            zB += __shfl_xor_sync(0xffffffffu, zB, o);
          }
          const size_t pbase = ((size_t)c * Hq + (size_t)h * G) * npt + part;
#pragma unroll
          for (int mt = 0; mt < T::MT; ++mt) {
            const int d0 = DS * gq + 2 * mt;
            if (realA) {
              float* o = d.po + (pbase + (size_t)hA * npt) * D;
              o[d0] = O[mt][0];
              o[d0 + 1] = O[mt][2];
            }
            if (realB) {
              float* o = d.po + (pbase + (size_t)hB * npt) * D;
              o[d0] = O[mt][1];
              o[d0 + 1] = O[mt][3];
            }
          }
          if (gq == 0) {
            if (realA) { d.pm[pbase + (size_t)hA * npt] = mA; d.pz[pbase + (size_t)hA * npt] = zA; }
            if (realB) { d.pm[pbase + (size_t)hB * npt] = mB; d.pz[pbase + (size_t)hB * npt] = zB; }
          }
          continue;
        }
      }
      uint32_t bn[T::KSTEPS][2];
      {
        const __half* qn = q + ((size_t)(c - c0) * Hq + (size_t)h * G + gq) * D + 2 * cq;
#pragma unroll
        for (int kk = 0; kk < T::KSTEPS; ++kk) {
          bn[kk][0] = gq < G ? *reinterpret_cast<const uint32_t*>(qn + 16 * kk) : 0u;
          bn[kk][1] = gq < G ? *reinterpret_cast<const uint32_t*>(qn + 16 * kk + 8) : 0u;
        }
      }
      float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.sld;
      float mA = -INFINITY, mB = -INFINITY, zA = 0.f, zB = 0.f;
      float O[T::MT][4];
#pragma unroll
      for (int mt = 0; mt < T::MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) O[mt][i] = 0.f;
      for (int t = 0; t < ntiles; ++t, ++gtile) {
        const int s = gtile % NSW;
        const uint32_t kb = sbase + (uint32_t)((warp * NSW + s) * T::SLOT), vb = kb + T::NSUB * T::SUB;
        mbar_wait(bar(T::B_FULL + warp * NSW + s), (gtile / NSW) & 1);
        const int tb = begin + t * TT;
        const int nvalid = min(TT, begin + ntok - tb);
        float ca[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
        for (int kk = 0; kk < T::KSTEPS; ++kk) {
          const int ch = 2 * kk + lc;
          uint32_t a[4];
          ldsm_x4(kb + (ch >> 3) * T::SUB + lr * 128 + (((ch & 7) ^ (lr & 7)) << 4), a);
          mma16816(ca[kk & 1], a, bn[kk][0], bn[kk][1]);
        }
        const int t0 = tb + gq, t1 = tb + gq + 8;
        const bool v0 = gq < nvalid, v1 = gq + 8 < nvalid;
        const float s0 = v0 ? (ca[0][0] + ca[1][0]) * qscale : -INFINITY;
        const float s1 = v0 ? (ca[0][1] + ca[1][1]) * qscale : -INFINITY;
        const float s2 = v1 ? (ca[0][2] + ca[1][2]) * qscale : -INFINITY;
        const float s3 = v1 ? (ca[0][3] + ca[1][3]) * qscale : -INFINITY;
        if (realA) {
          if (v0) scoreg[(size_t)hA * d.sld + t0] = s0;
          if (v1) scoreg[(size_t)hA * d.sld + t1] = s2;
        }
        if (realB) {
          if (v0) scoreg[(size_t)hB * d.sld + t0] = s1;
          if (v1) scoreg[(size_t)hB * d.sld + t1] = s3;
        }
        float tA = fmaxf(s0, s2), tB = fmaxf(s1, s3);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          tA = fmaxf(tA, __shfl_xor_sync(0xffffffffu, tA, o));
          tB = fmaxf(tB, __shfl_xor_sync(0xffffffffu, tB, o));
        }
        const float nA = fmaxf(mA, tA), nB = fmaxf(mB, tB);
        const float cA = (mA == nA) ? 1.f : expf(mA - nA), cB = (mB == nB) ? 1.f : expf(mB - nB);
        const float p0 = (v0 && realA) ? expf(s0 - nA) : 0.f, p2 = (v1 && realA) ? expf(s2 - nA) : 0.f;
        const float p1 = (v0 && realB) ? expf(s1 - nB) : 0.f, p3 = (v1 && realB) ? expf(s3 - nB) : 0.f;
        zA = zA * cA + (p0 + p2);
        zB = zB * cB + (p1 + p3);
        mA = nA;
        mB = nB;
        {
          const __half h0 = __float2half_rn(p0), h1 = __float2half_rn(p1);
          const __half h2 = __float2half_rn(p2), h3 = __float2half_rn(p3);
          sPh[hA * TT + gq] = __half_as_ushort(h0);
          sPh[hA * TT + gq + 8] = __half_as_ushort(h2);
          sPh[hB * TT + gq] = __half_as_ushort(h1);
          sPh[hB * TT + gq + 8] = __half_as_ushort(h3);
          sPl[hA * TT + gq] = __half_as_ushort(__float2half_rn(p0 - __half2float(h0)));
          sPl[hA * TT + gq + 8] = __half_as_ushort(__float2half_rn(p2 - __half2float(h2)));
          sPl[hB * TT + gq] = __half_as_ushort(__float2half_rn(p1 - __half2float(h1)));
          sPl[hB * TT + gq + 8] = __half_as_ushort(__float2half_rn(p3 - __half2float(h3)));
        }
        if (cA != 1.f || cB != 1.f) {
#pragma unroll
          for (int mt = 0; mt < T::MT; ++mt) {
            O[mt][0] *= cA; O[mt][1] *= cB; O[mt][2] *= cA; O[mt][3] *= cB;
          }
        }
        __syncwarp();
        const uint32_t ph0 = *reinterpret_cast<const uint32_t*>(sPh + gq * TT + 2 * cq);
        const uint32_t ph1 = *reinterpret_cast<const uint32_t*>(sPh + gq * TT + 2 * cq + 8);
        const uint32_t pl0 = *reinterpret_cast<const uint32_t*>(sPl + gq * TT + 2 * cq);
        const uint32_t pl1 = *reinterpret_cast<const uint32_t*>(sPl + gq * TT + 2 * cq + 8);
#pragma unroll
        for (int mt = 0; mt < T::MT; ++mt) {
          const int ch = 2 * mt + vc;
          uint32_t a[4];
          ldsm_x4_t(vb + (ch >> 3) * T::SUB + vr * 128 + (((ch & 7) ^ (vr & 7)) << 4), a);
          mma16816(O[mt], a, ph0, ph1);
          mma16816(O[mt], a, pl0, pl1);
        }
        __syncwarp();                                   // slot and sP reads done
        if (lane == 0) mbar_arrive(bar(T::B_EMPTY + warp * NSW + s));
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        zA += __shfl_xor_sync(0xffffffffu, zA, o);
        zB += __shfl_xor_sync(0xffffffffu, zB, o);
      }
      // the unit's partial slot: (m, z) per head, O in natural dim order
      const size_t pbase = ((size_t)c * Hq + (size_t)h * G) * npt + part;
#pragma unroll
      for (int mt = 0; mt < T::MT; ++mt) {
        const int d0 = 16 * mt + gq;
        if (realA) {
          float* o = d.po + (pbase + (size_t)hA * npt) * D;
          o[d0] = O[mt][0];
          o[d0 + 8] = O[mt][2];
        }
        if (realB) {
          float* o = d.po + (pbase + (size_t)hB * npt) * D;
          o[d0] = O[mt][1];
          o[d0 + 8] = O[mt][3];
        }
      }
      if (gq == 0) {
        if (realA) { d.pm[pbase + (size_t)hA * npt] = mA; d.pz[pbase + (size_t)hA * npt] = zA; }
        if (realB) { d.pm[pbase + (size_t)hB * npt] = mB; d.pz[pbase + (size_t)hB * npt] = zB; }
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // the caller's TMA may overwrite what we read
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < T::N_BAR; ++i) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar(i)) : "memory");
  __syncthreads();
}

template <int D, int G>
__global__ void __launch_bounds__(TsP<D, G>::THREADS, D == 128 ? 2 : 3)
k2_fp16_stream(Dev d, const __grid_constant__ Maps maps, int c0, int ccount, const __half* __restrict__ q,
               float qscale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  asm volatile("griddepcontrol.launch_dependents;");
  CKV_TL(3, 0);
  fp16_units<D, G>(d, maps, c0, ccount, q, qscale, smem);
  CKV_TL(3, 2);
  // completes only after its programmatic prerequisite (the general kernel), so the grids
  // launched after this one see every partial
  asm volatile("griddepcontrol.wait;" ::: "memory");
}


// Combine split partials -> out; normalised weights -> head mean (fp64) -> abar.
template <int D, int G, bool BULK = true>
__global__ void __launch_bounds__(kMmaWarps * 32, 3)
k2_attend_mma(Dev d, const __grid_constant__ Maps maps, int c0, const __half* __restrict__ q, float qscale,
              int skip_bulk) {
  using T = TrM<D, G>;
  extern __shared__ __align__(1024) uint8_t smem[];
  // let the tcgen05 persistent grid (a programmatic dependent sharing no data) start beside us
  asm volatile("griddepcontrol.launch_dependents;");
  const int c = c0 + blockIdx.z, h = blockIdx.y;
  CKV_TL(0, 0);
  if (!skip_bulk) {
    const int n = d.len[c], nq = d.nq[c];
    int b, e;
    part_range(d, blockIdx.x, 0, n, nq, b, e);
    // single-segment codes parts run on the streaming kernel when it takes them (d.scodes)
    if (d.scodes && b < e && __ldg(d.seg + (size_t)c * d.cap + b) == __ldg(d.seg + (size_t)c * d.cap + e - 1)) return;
    mma_split<D, G, BULK>(d, maps, c0, q, qscale, c, h, b, e, 2 * blockIdx.x, smem);
    return;
  }
  // Single-segment codes parts belong to the tcgen05 kernel. Work units are (cache, KV head,
  // j < gen_w) over the launch's `ncache` caches; unit (pair, j) runs the j-th, (j+gen_w)-th,
  // ... of the pair's other non-empty parts (FP16 parts, multi-segment codes parts), in order.
  // The grid is either one unit per CTA (gen_w = the host's estimate of general splits per
  // cache) or smaller with CTAs looping over units (launch_split).
  int* s_list = reinterpret_cast<int*>(smem + T::OFF_X);
  __shared__ int s_cnt, s_pre;
  const int lane = threadIdx.x & 31;
  const uint32_t bars = smem_u32(smem) + T::OFF_BAR + 8 * 8 * (threadIdx.x >> 5);
  const int gen_w = max(1, d.gen_splits);
  const int units = skip_bulk * d.Hkv * gen_w;   // skip_bulk = the launch's cache count
  if (d.scodes) {
    // capped grid (see launch_split): one round trip for all of this CTA's units -- a pair has
    // work here only with two lossy segments in use
    bool any = false;
    for (int u = blockIdx.x + threadIdx.x * gridDim.x; u < units; u += blockDim.x * gridDim.x)
      any |= d.smax - __ldg(d.stop + c0 + (u / gen_w) / d.Hkv) >= 2;
    if (!__syncthreads_or(any)) return;
  }
  bool first = true, first_of_pair = false;
  int have = -1;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int pair = u / gen_w, j = u - pair * gen_w;
    const int pc = c0 + pair / d.Hkv, ph = pair % d.Hkv;
    // with the FP16 parts on the streaming kernel, a pair has work here only if some codes part
    // spans two lossy segments, which takes two lossy segments in use (smax - stop, kept by K3):
    // the bulk steady state has one, so its 2,048 CTAs exit here (14.5 -> ~2 us)
    if (d.fstream && d.smax - __ldg(d.stop + pc) < 2) continue;
    if (pair != have) {
      __syncthreads();   // the previous pair's list is no longer read
      if (threadIdx.x >= 32 && d.fstream) {
        if (threadIdx.x == 32) s_pre = -1;     // FP16 parts run on the streaming kernel
      } else if (threadIdx.x >= 32) {
        // beside the list (warp 0), warps 1-3 stage the slot rows of the pair's last FP16 part
        // (in the bulk steady state the only general part): one dependent round trip less
        const int n = d.len[pc], nq = d.nq[pc];
        const int np2 = (n + kSplitTokens - 1) / kSplitTokens;
        int b = 0, e = 0;
        for (int sp = np2 - 1; sp >= 0 && b >= e; --sp) part_range(d, sp, 1, n, nq, b, e);
        if (b < e && e - b <= kSplitTokens + kAbsorbTokens) {
          const size_t cb = (size_t)pc * d.cap;
          int* s_row = reinterpret_cast<int*>(smem + T::OFF_ROW);
          for (int j = threadIdx.x - 32; j < e - b; j += kMmaWarps * 32 - 32)
            s_row[j] = (int)((cb + __ldg(d.slot + cb + b + j)) * d.Hkv + ph);
          if (threadIdx.x == 32) s_pre = b;
        } else if (threadIdx.x == 32) {
          s_pre = -1;
        }
      }
      if (threadIdx.x < 32) {
        const int n = d.len[pc], nq = d.nq[pc];
        const int np = 2 * ((n + kSplitTokens - 1) / kSplitTokens);
        int cnt = 0;
        for (int b0 = 0; b0 < np; b0 += 32) {
          const int p = b0 + lane;
          bool gen = false;
          if (p < np) {
            int b, e;
            part_range(d, p >> 1, p & 1, n, nq, b, e);
            gen = b < e && ((p & 1) ? !d.fstream
                                    : __ldg(d.seg + (size_t)pc * d.cap + b) != __ldg(d.seg + (size_t)pc * d.cap + e - 1));
          }
          const unsigned m = __ballot_sync(0xffffffffu, gen);
          if (gen) s_list[cnt + __popc(m & ((1u << lane) - 1u))] = p;
          cnt += __popc(m);
        }
        if (lane == 0) s_cnt = cnt;
      }
      __syncthreads();
      have = pair;
      first_of_pair = true;
    }
    const int cnt = s_cnt;
    for (int idx = j; idx < cnt; idx += gen_w) {
      if (!first) {   // re-arm this warp's barriers for the next split
        __syncthreads();
        if (lane == 0)
          for (int s = 0; s < 8; ++s) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bars + 8 * s) : "memory");
        __syncthreads();
      }
      first = false;
      const int p = s_list[idx];
      int b, e;
      part_range(d, p >> 1, p & 1, d.len[pc], d.nq[pc], b, e);
      // staged rows are valid for the first part run after the list only (mma_split reuses them)
      const bool staged = first_of_pair && (p & 1) && b == s_pre && b >= d.nq[pc];
      first_of_pair = false;
      mma_split<D, G, BULK>(d, maps, c0, q, qscale, pc, ph, b, e, p, smem, staged);
    }
  }
  CKV_TL(0, 2);
}

constexpr int kCombThreads = 256;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// (double)w for a weight from ex2f (+0, a normal positive float, or NaN) on the integer pipes:
// F2F.F64.F32 issues on the same quarter-rate XU pipe as MUFU.EX2, which the head-mean loop
// saturates. Exact: rebias the exponent (127 -> 1023) and move the 23-bit mantissa up 29 bits.
__device__ __forceinline__ double w2d(float w) {
  const uint32_t u = __float_as_uint(w);
  const uint32_t hi0 = (u >> 3) + 0x38000000u;
  const uint32_t sp = u ? 0x7ff80000u : 0u;            // +0 -> +0.0; inf / NaN -> NaN
  const uint32_t hi = (u - 1u < 0x7f7fffffu) ? hi0 : sp;
  return __hiloint2double((int)hi, (int)(u << 29));
}

// Split merge + EMA staging for one chunk of EPT * kCombThreads entries of one cache (EPT
// consecutive entries per thread: 4 = one float4 of scores per head for big grids, 1 for the
// few-cache launches of a per-layer decode forward, where 4x more CTAs shorten the tail).
// Latency: the first heads' score loads are issued before anything else; the per-head split
// statistics are reduced with lanes = partial slots (4 heads per warp, all loads in flight,
// shuffle max / sum). Issue: each normalised weight is one FFMA + one EX2,
// w = 2^(s*log2e - (M*log2e + log2 Z)), with the per-head offset precomputed in shared
// memory; whole 8/16-head chunks run without per-head bounds checks; the weights dump is a
// separate instantiation. The output merge reads float4s of 4 dims with 8 partials in flight.
template <int EPT, bool WD>
__global__ void __launch_bounds__(kCombThreads, EPT == 4 ? 3 : 4)
k2_combine(Dev d, int c0, float* __restrict__ out, float* __restrict__ wdump, int D) {
  CKV_TL(2, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // inline K1 (hence every attention grid) done
  constexpr int HF = EPT == 4 ? 8 : 16;   // heads' score loads in flight per thread
  constexpr float kLog2e = 1.4426950408889634f;
  extern __shared__ float sm[];
  const int Hq = d.Hq, nsp = d.npart;
  float* sM = sm;                 // [Hq]
  float* sZ = sM + Hq;            // [Hq]
  float* sR = sZ + Hq;            // [Hq] M*log2e + log2 Z (exponent offset)
  float* sF = sR + Hq;            // [Hq][npart] rescale factors (0 for empty parts)
  const int c = c0 + blockIdx.y;
  const int n = d.len[c], nq = d.nq[c];
  const int nused = 2 * ((n + kSplitTokens - 1) / kSplitTokens);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = (blockIdx.x * kCombThreads + threadIdx.x) * EPT;
  const bool has_ent = i < n;
  const float* sp = d.score + (size_t)c * Hq * d.sld + i;
  const size_t sld = d.sld;
  float v[HF][EPT];
  auto load = [&](int k, const float* p) {
    if constexpr (EPT == 4) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(p));
      v[k][0] = x.x; v[k][1] = x.y; v[k][2] = x.z; v[k][3] = x.w;
    } else {
      v[k][0] = __ldg(p);
    }
  };
  if (has_ent && Hq >= HF) {
#pragma unroll
    for (int k = 0; k < HF; ++k) load(k, sp + k * sld);
  }
  if (nused <= 32) {
    int pb, pe;
    part_range(d, lane >> 1, lane & 1, n, nq, pb, pe);
    const bool live = lane < nused && pb < pe;   // empty parts are never written
    for (int g0 = warp; g0 < Hq; g0 += 4 * (kCombThreads / 32)) {
      float pm[4], pz[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int g = g0 + j * (kCombThreads / 32);
        const size_t pi = ((size_t)c * Hq + g) * nsp + lane;
        pm[j] = (g < Hq && live) ? __ldg(d.pm + pi) : -INFINITY;
        pz[j] = (g < Hq && live) ? __ldg(d.pz + pi) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int g = g0 + j * (kCombThreads / 32);
        float M = pm[j];
#pragma unroll
        for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float f = (pm[j] == -INFINITY) ? 0.f : expf(pm[j] - M);
        float Z = f * pz[j];
#pragma unroll
        for (int o = 16; o; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
        if (g < Hq) {
          if (lane < nused) sF[g * nsp + lane] = f;
          if (lane == 0) {
            sM[g] = M;
            sZ[g] = Z;
            sR[g] = Z > 0.f ? fmaf(M, kLog2e, __log2f(Z)) : INFINITY;
          }
        }
      }
    }
  } else {
    for (int g = threadIdx.x; g < Hq; g += blockDim.x) {
      const size_t pi = ((size_t)c * Hq + g) * nsp;
      float M = -INFINITY;
      for (int s = 0; s < nused; ++s) {
        int pb, pe;
        part_range(d, s >> 1, s & 1, n, nq, pb, pe);
        const float pm = pb < pe ? __ldg(d.pm + pi + s) : -INFINITY;
        sF[g * nsp + s] = pm;
        M = fmaxf(M, pm);
      }
      float Z = 0.f;
      for (int s = 0; s < nused; ++s) {
        const float pm = sF[g * nsp + s];
        const float f = (pm == -INFINITY) ? 0.f : expf(pm - M);
        sF[g * nsp + s] = f;
        if (f != 0.f) Z += f * __ldg(d.pz + pi + s);
      }
      sM[g] = M;
      sZ[g] = Z;
      sR[g] = Z > 0.f ? fmaf(M, kLog2e, __log2f(Z)) : INFINITY;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = n;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *d.work = 0;   // next K2 launch
  // Head mean of the normalised weights w = exp(s - M) / Z of this thread's entries; each
  // entry's fp64 chain sums heads strictly in head order (NumPy's axis-0 reduction order) and
  // divides by Hq.
  if (has_ent) {
    double a[EPT];
#pragma unroll
    for (int j = 0; j < EPT; ++j) a[j] = 0.0;
    auto consume = [&](int k, int g) {
      const float off = sR[g];
      float w[EPT];
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        w[j] = ex2f(fmaf(v[k][j], kLog2e, -off));
        a[j] = __dadd_rn(a[j], (double)w[j]);
      }
      if constexpr (WD) {
        float* wp = wdump + ((size_t)(c - c0) * Hq + g) * d.cap + i;
#pragma unroll
        for (int j = 0; j < EPT; ++j)
          if (i + j < n) wp[j] = w[j];
      }
    };
    int g0 = 0;
    for (; g0 + HF <= Hq; g0 += HF) {   // whole chunks, no per-head checks
      if (g0) {
#pragma unroll
        for (int k = 0; k < HF; ++k) load(k, sp + (size_t)(g0 + k) * sld);
      }
#pragma unroll
      for (int k = 0; k < HF; ++k) consume(k, g0 + k);
    }
    for (int g = g0; g < Hq; ++g) {     // tail heads
      load(0, sp + (size_t)g * sld);
      consume(0, g);
    }
    const double hq = (double)Hq;
    double* ab = d.abar + (size_t)c * d.cap + i;
#pragma unroll
    for (int j = 0; j < EPT; ++j)
      if (i + j < n) ab[j] = __ddiv_rn(a[j], hq);
  }
  if (out) {
    // every block of the cache merges a slice of the Hq*D outputs, 4 dims (one float4) per
    // thread and 8 partials in flight
    const int nq4 = Hq * D / 4;
    const int per_o = (nq4 + gridDim.x - 1) / gridDim.x;
    const int o1 = min(nq4, (blockIdx.x + 1) * per_o);
    for (int idx = blockIdx.x * per_o + threadIdx.x; idx < o1; idx += blockDim.x) {
      const int e0 = 4 * idx;
      const int g = e0 / D, dd = e0 - g * D;
      const float4* pp = reinterpret_cast<const float4*>(d.po + ((size_t)c * Hq + g) * nsp * D + dd);
      const float* fg = sF + g * nsp;
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < nused; s0 += 8) {
        float4 pv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          pv[k] = (s0 + k < nused && fg[s0 + k] != 0.f) ? __ldg(pp + (size_t)(s0 + k) * (D / 4))
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float f = s0 + k < nused ? fg[s0 + k] : 0.f;
          o.x = fmaf(f, pv[k].x, o.x); o.y = fmaf(f, pv[k].y, o.y);
          o.z = fmaf(f, pv[k].z, o.z); o.w = fmaf(f, pv[k].w, o.w);
        }
      }
      const float z = sZ[g];
      const float rz = z > 0.f ? 1.f / z : 0.f;
      float4 r = make_float4(o.x * rz, o.y * rz, o.z * rz, o.w * rz);
      if (!(z > 0.f)) r = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(out + ((size_t)(c - c0) * Hq + g) * D + dd) = r;
    }
  }
  CKV_TL(2, 2);
}

// Staged variant of k2_combine for big launches (all layers): one CTA per 1,024 entries of a
// cache. The EMA head mean's score reads were latency-bound in registers (8 heads in flight per
// thread, one HBM round trip per 8 heads); here one thread streams the CTA's [Hq][1024] score
// block into a 2-stage shared-memory ring of 8-head chunks with bulk copies (32 KB in flight per
// stage, no registers held), and the split-partial output merge runs while the first chunks land.
constexpr int kCombHeads = 8;                         // heads per staged chunk
constexpr int kCombEnt = 4 * kCombThreads;            // entries per CTA
constexpr int kCombStageBytes = kCombHeads * kCombEnt * 4;
constexpr int kCombRing = 2 * kCombStageBytes;

template <bool WD>
__global__ void __launch_bounds__(kCombThreads, 3)
k2_combine_staged(Dev d, int c0, float* __restrict__ out, float* __restrict__ wdump, int D) {
  CKV_TL(2, 0);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // inline K1 (hence every attention grid) done
  constexpr float kLog2e = 1.4426950408889634f;
  extern __shared__ __align__(128) uint8_t csm[];
  const uint32_t ring = smem_u32(csm);
  const uint32_t bars = ring + kCombRing;
  const int Hq = d.Hq, nsp = d.npart;
  float* sM = reinterpret_cast<float*>(csm + kCombRing + 16);   // [Hq]
  float* sZ = sM + Hq;            // [Hq]
  float* sR = sZ + Hq;            // [Hq] M*log2e + log2 Z (exponent offset)
  float* sF = sR + Hq;            // [Hq][npart] rescale factors (0 for empty parts)
  const int c = c0 + blockIdx.y;
  const int n = d.len[c], nq = d.nq[c];
  const int nused = 2 * ((n + kSplitTokens - 1) / kSplitTokens);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.x * kCombEnt;
  const int ne = min(n - i0, kCombEnt);                 // entries of this CTA (may be <= 0)
  const int nch = (Hq + kCombHeads - 1) / kCombHeads;
  const uint32_t rowb = ne > 0 ? (uint32_t)(((ne + 3) & ~3) * 4) : 0u;
  const float* srow = d.score + (size_t)c * Hq * d.sld + i0;
  auto issue = [&](int k) {   // chunk k (heads 8k..) -> stage k % 2
    const int st = k & 1, h0 = k * kCombHeads, nh = min(kCombHeads, Hq - h0);
    const uint32_t bar = bars + 8 * st;
    mbar_arrive_tx(bar, (uint32_t)nh * rowb);
    for (int hh = 0; hh < nh; ++hh)
      tma_row(ring + st * kCombStageBytes + hh * kCombEnt * 4, srow + (size_t)(h0 + hh) * d.sld, rowb, bar);
  };
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (ne > 0) {
      issue(0);
      if (nch > 1) issue(1);
    }
  }
  // per-head split statistics (lanes = partial slots)
  if (nused <= 32) {
    int pb, pe;
    part_range(d, lane >> 1, lane & 1, n, nq, pb, pe);
    const bool live = lane < nused && pb < pe;   // empty parts are never written
    for (int g0 = warp; g0 < Hq; g0 += 4 * (kCombThreads / 32)) {
      float pm[4], pz[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int g = g0 + j * (kCombThreads / 32);
        const size_t pi = ((size_t)c * Hq + g) * nsp + lane;
        pm[j] = (g < Hq && live) ? __ldg(d.pm + pi) : -INFINITY;
        pz[j] = (g < Hq && live) ? __ldg(d.pz + pi) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int g = g0 + j * (kCombThreads / 32);
        float M = pm[j];
#pragma unroll
        for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        const float f = (pm[j] == -INFINITY) ? 0.f : expf(pm[j] - M);
        float Z = f * pz[j];
#pragma unroll
        for (int o = 16; o; o >>= 1) Z += __shfl_xor_sync(0xffffffffu, Z, o);
        if (g < Hq) {
          if (lane < nused) sF[g * nsp + lane] = f;
          if (lane == 0) {
            sM[g] = M;
            sZ[g] = Z;
            sR[g] = Z > 0.f ? fmaf(M, kLog2e, __log2f(Z)) : INFINITY;
          }
        }
      }
    }
  } else {
    for (int g = threadIdx.x; g < Hq; g += blockDim.x) {
      const size_t pi = ((size_t)c * Hq + g) * nsp;
      float M = -INFINITY;
      for (int s = 0; s < nused; ++s) {
        int pb, pe;
        part_range(d, s >> 1, s & 1, n, nq, pb, pe);
        const float pm = pb < pe ? __ldg(d.pm + pi + s) : -INFINITY;
        sF[g * nsp + s] = pm;
        M = fmaxf(M, pm);
      }
      float Z = 0.f;
      for (int s = 0; s < nused; ++s) {
        const float pm = sF[g * nsp + s];
        const float f = (pm == -INFINITY) ? 0.f : expf(pm - M);
        sF[g * nsp + s] = f;
        if (f != 0.f) Z += f * __ldg(d.pz + pi + s);
      }
      sM[g] = M;
      sZ[g] = Z;
      sR[g] = Z > 0.f ? fmaf(M, kLog2e, __log2f(Z)) : INFINITY;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = n;
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *d.work = 0;   // next K2 launch
  if (out) {
    // every block of the cache merges a slice of the Hq*D outputs (one float4 of 4 dims per
    // thread, 8 partials in flight) while its score chunks stream in
    const int nq4 = Hq * D / 4;
    const int per_o = (nq4 + gridDim.x - 1) / gridDim.x;
    const int o1 = min(nq4, (blockIdx.x + 1) * per_o);
    for (int idx = blockIdx.x * per_o + threadIdx.x; idx < o1; idx += blockDim.x) {
      const int e0 = 4 * idx;
      const int g = e0 / D, dd = e0 - g * D;
      const float4* pp = reinterpret_cast<const float4*>(d.po + ((size_t)c * Hq + g) * nsp * D + dd);
      const float* fg = sF + g * nsp;
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int s0 = 0; s0 < nused; s0 += 8) {
        float4 pv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          pv[k] = (s0 + k < nused && fg[s0 + k] != 0.f) ? __ldg(pp + (size_t)(s0 + k) * (D / 4))
                                                        : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float f = s0 + k < nused ? fg[s0 + k] : 0.f;
          o.x = fmaf(f, pv[k].x, o.x); o.y = fmaf(f, pv[k].y, o.y);
          o.z = fmaf(f, pv[k].z, o.z); o.w = fmaf(f, pv[k].w, o.w);
        }
      }
      const float z = sZ[g];
      const float rz = z > 0.f ? 1.f / z : 0.f;
      float4 r = make_float4(o.x * rz, o.y * rz, o.z * rz, o.w * rz);
      if (!(z > 0.f)) r = make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(out + ((size_t)(c - c0) * Hq + g) * D + dd) = r;
    }
  }
  CKV_TL(2, 1);   // statistics + output merge done
  if (ne <= 0) {
    CKV_TL(2, 2);
    return;
  }
  // Head mean of the normalised weights w = exp(s - M) / Z of this thread's 4 entries; each
  // entry's fp64 chain sums heads strictly in head order (NumPy's axis-0 reduction order) and
  // divides by Hq.
  const int e = 4 * threadIdx.x;
  const bool has_ent = e < ne;
  double a[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < nch; ++k) {
    const int st = k & 1, h0 = k * kCombHeads, nh = min(kCombHeads, Hq - h0);
    mbar_wait(bars + 8 * st, (k >> 1) & 1);
    if (has_ent) {
      const float* sb = reinterpret_cast<const float*>(csm + st * kCombStageBytes) + e;
      for (int hh = 0; hh < nh; ++hh) {
        const float4 x = *reinterpret_cast<const float4*>(sb + hh * kCombEnt);
        const float off = sR[h0 + hh];
        const float w[4] = {ex2f(fmaf(x.x, kLog2e, -off)), ex2f(fmaf(x.y, kLog2e, -off)),
                            ex2f(fmaf(x.z, kLog2e, -off)), ex2f(fmaf(x.w, kLog2e, -off))};
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = __dadd_rn(a[j], w2d(w[j]));
        if constexpr (WD) {
          float* wp = wdump + ((size_t)(c - c0) * Hq + h0 + hh) * d.cap + i0 + e;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (e + j < ne) wp[j] = w[j];
        }
      }
    }
    __syncthreads();                                   // stage st consumed
    if (threadIdx.x == 0 && k + 2 < nch) issue(k + 2);
  }
  if (has_ent) {
    const double hq = (double)Hq;
    double* ab = d.abar + (size_t)c * d.cap + i0 + e;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (e + j < ne) ab[j] = __ddiv_rn(a[j], hq);
  }
  CKV_TL(2, 2);
}

// Parity hook: head mean of host-supplied fp64 rows (update_attention_ema input). A row block
// must have exactly valid_len entries (cache.py:164-167): ld == n, or ld > n with the caller's
// NaN pad at column n (ragged per-sequence rows); otherwise nothing is staged and the step
// reports kStShape (ValueError).
__global__ void k2_stage_rows(Dev d, int layer, const double* __restrict__ rows, int ld) {
  const int b = blockIdx.y;
  const int c = layer * d.B + b;
  const int n = d.len[c];
  const int Hq = d.Hq;
  const bool ok = ld == n || (ld > n && isnan(rows[(size_t)b * Hq * ld + n]));
  if (!ok) {
    if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = -2;
    return;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int g = 0; g < Hq; ++g) a = __dadd_rn(a, rows[((size_t)b * Hq + g) * ld + i]);
    d.abar[(size_t)c * d.cap + i] = __ddiv_rn(a, (double)Hq);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = n;
}

// Head-sharded EMA input: the attention weights of every head shard, all-gathered as
// [shards][ccount][Hq_local][cap] fp32, summed in global head order (shard-major, the
// order a single-GPU run sums them) in fp64 and divided by the total head count.
__global__ void k2_stage_weights(Dev d, int c0, int ccount, const float* __restrict__ w, int shards) {
  const int c = c0 + blockIdx.y;
  const int n = d.len[c];
  const int Hql = d.Hq;
  const double htot = (double)(Hql * shards);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int r = 0; r < shards; ++r)
      for (int g = 0; g < Hql; ++g)
        a = __dadd_rn(a, (double)__ldg(w + (((size_t)r * ccount + (c - c0)) * Hql + g) * d.cap + i));
    d.abar[(size_t)c * d.cap + i] = __ddiv_rn(a, htot);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = n;
}

// Head-sharded EMA input as a chain in global head order: shard r continues shard r-1's fp64
// running head sum (acc_in, NULL for shard 0) over its own heads in order, reading its
// ckv_attend weights dump [ccount caches][Hq_local][cap]; the last shard's sum is
// the single-GPU sum bit for bit (NumPy's sequential axis-0 reduction, cache.py:171).
__global__ void k2_head_partial(Dev d, int c0, const float* __restrict__ w, const double* __restrict__ acc_in,
                                double* __restrict__ acc_out) {
  const int c = c0 + blockIdx.y;
  const int n = d.len[c];
  const int Hql = d.Hq;
  const size_t ab = (size_t)(c - c0) * d.cap;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = acc_in ? acc_in[ab + i] : 0.0;
    for (int g = 0; g < Hql; ++g) a = __dadd_rn(a, (double)__ldg(w + ((size_t)(c - c0) * Hql + g) * d.cap + i));
    acc_out[ab + i] = a;
  }
}

// ... and every shard stages mean = sum / total heads (update_attention_ema's `mean`).
__global__ void k2_stage_mass(Dev d, int c0, const double* __restrict__ acc, int total_heads) {
  const int c = c0 + blockIdx.y;
  const int n = d.len[c];
  const double ht = (double)total_heads;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    d.abar[(size_t)c * d.cap + i] = __ddiv_rn(acc[(size_t)(c - c0) * d.cap + i], ht);
  if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = n;
}

template <int D, int G>
cudaError_t launch_split(const Dev& d, const Maps& maps, int c0, int ccount, const __half* q, cudaStream_t s) {
  dim3 grid(d.live_splits, d.Hkv, ccount);
  const float qs = (float)(1.0 / sqrt((double)D));
  static bool configured = false;
  if constexpr (D >= 64) {
    using T = TrM<D, G>;
    using TS = TsP<D, G>;
    static int nsm = 0;
    if (!configured) {
      cudaError_t e = cudaFuncSetAttribute(k2_attend_mma<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k2_attend_mma<D, G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k2_fp16_stream<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, TS::SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k2_fp16_stream<D, G>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
      if constexpr (D == 128) {
        e = cudaFuncSetAttribute(k2_i8_persistent<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcP<G>::SMEM);
        if (e != cudaSuccess) return e;
      }
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      configured = true;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    // Codes parts (cut mode) / mixed splits: the general kernel, launched first. With the tcgen05
    // grid on, it runs one CTA per (cache, head, j < gen_splits) unit over the pairs' multi-segment
    // codes parts (and FP16 parts when the streaming kernel is off); otherwise one CTA per split.
    bool chained = false;
    if (d.cut_nq && ((d.use_tc && kTcEnabled && D == 128) || (d.scodes && d.gen_cap))) {
      int gen_ctas = ccount * d.Hkv * std::max(1, d.gen_splits);
      // Without the tcgen05 grid the streaming kernel takes the single-segment codes parts too, so
      // only multi-segment codes parts are left here: one wave of CTAs loops over the units, each
      // CTA testing all of its units with one load round trip (Qwen-32B pyramid: 8,192 one-load
      // CTAs, ~12.5 us before the stream started -> one wave: 223.7 -> 214.1 us/step). Beside the
      // tcgen05 grid the same cap was slower (INT8 4K 484 -> 488 us), so there it stays off.
      // CKV_GENCAP=0 restores the per-split grid.
      if (d.scodes && d.gen_cap) gen_ctas = std::min(gen_ctas, 2 * nsm);
      k2_attend_mma<D, G, false><<<gen_ctas, kMmaWarps * 32, T::SMEM, s>>>(d, maps, c0, q, qs, ccount);
      ++g_k2_launches;
      chained = true;
    } else if (d.quant || !d.fstream) {
      if (d.quant) k2_attend_mma<D, G><<<grid, kMmaWarps * 32, T::SMEM, s>>>(d, maps, c0, q, qs, 0);
      else k2_attend_mma<D, G, false><<<grid, kMmaWarps * 32, T::SMEM, s>>>(d, maps, c0, q, qs, 0);   // no codes
      ++g_k2_launches;
      chained = true;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (d.fstream) {
      // FP16 parts: the persistent streaming kernel, the general kernel's programmatic dependent
      // (its CTAs take SM room as the general kernel's CTAs retire)
      const int units = ccount * d.Hkv * d.live_splits;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(std::max(1, std::min((D == 128 ? 2 : 3) * nsm, units)));
      cfg.blockDim = dim3(TS::THREADS);
      cfg.dynamicSmemBytes = TS::SMEM;
      cfg.stream = s;
      cfg.attrs = attr;
      cfg.numAttrs = chained ? 1 : 0;
      e = cudaLaunchKernelEx(&cfg, k2_fp16_stream<D, G>, d, maps, c0, ccount, q, qs);
      ++g_k2_launches;
      if (e != cudaSuccess) return e;
      chained = true;
    }
    if constexpr (D == 128 && kTcEnabled) {
      if (d.cut_nq && d.use_tc) {
        // the single-segment INT8 splits: the persistent tcgen05 kernel (2 CTAs per SM), the
        // previous grid's programmatic dependent
        const int items = ccount * d.Hkv * d.live_splits;
        Dev dp = d;
        dp.dyn_items = items < 8 * 2 * nsm ? 1 : 0;
        if (d.dyn_force >= 0) dp.dyn_items = d.dyn_force;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(std::min(2 * nsm, items));
        cfg.blockDim = dim3(TcP<G>::THREADS);
        cfg.dynamicSmemBytes = TcP<G>::SMEM;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = chained ? 1 : 0;
        ++g_k2_launches;
        return cudaLaunchKernelEx(&cfg, k2_i8_persistent<G>, dp, maps, c0, ccount, q, qs);
      }
    }
  } else {
    using T = Tr<D, G>;
    if (!configured) {
      cudaError_t e = cudaFuncSetAttribute(k2_attend_split<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    k2_attend_split<D, G><<<grid, kThreads, T::SMEM, s>>>(d, maps, c0, q, qs);
    ++g_k2_launches;
  }
  return cudaGetLastError();
}

template <int D>
cudaError_t dispatch_g(const Dev& d, const Maps& maps, int c0, int ccount, const __half* q, cudaStream_t s) {
  switch (d.G) {
    case 1: return launch_split<D, 1>(d, maps, c0, ccount, q, s);
    case 2: return launch_split<D, 2>(d, maps, c0, ccount, q, s);
    case 4: return launch_split<D, 4>(d, maps, c0, ccount, q, s);
    case 5: return launch_split<D, 5>(d, maps, c0, ccount, q, s);
    case 8: return launch_split<D, 8>(d, maps, c0, ccount, q, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

int last_attend_launches() { return g_k2_launches; }

bool attend_supported(int D, int G) {
  const bool dok = D == 16 || D == 32 || D == 64 || D == 128;
  const bool gok = G == 1 || G == 2 || G == 4 || G == 5 || G == 8;
  return dok && gok;
}

cudaError_t launch_attend(const Dev& d0, const Maps& maps, int c0, int ccount, const __half* q,
                          float* out, float* wdump, cudaStream_t s, cudaEvent_t mid, K1Inline* k1) {
  Dev d = d0;
  // FP16 parts on the streaming kernel (D = 64 / 128; CKV_FSTREAM=0 keeps them on the general kernel)
  // Measured (r02, graph-replayed steps, big launches only): beside the tcgen05 grid (INT8 bulk
  // steady state: K2 458 -> 443 us), on FP16-only caches of >= 4 splits (Llama-8B FP16 4K: 737 ->
  // 726-736 us), and -- taking the single-segment codes parts too (d.scodes) -- on short INT8
  // caches without the tcgen05 grid (Qwen-32B pyramid, <= 2 splits: 218 -> 181 us). Long INT8
  // caches without it (decode-built 4K: 747 -> 780 us) and small launches (GPT-2, NIAH decode)
  // keep the general kernel. CKV_FSTREAM=0 / 1 forces it off / on (where D allows).
  const int fs_env = d.fs_force;   // CKV_FSTREAM at ckv_create
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const bool tc_launch = kTcEnabled && d.D == 128 && d.quant && d.use_tc;
  const bool big_launch = (long)ccount * d.Hkv * d.live_splits >= 8L * 2 * nsm;   // >= 8 items per persistent CTA
  d.fstream = d.D >= 64 && (fs_env == 1 || (fs_env < 0 && big_launch && (tc_launch || (!d.quant && d.live_splits >= 4) ||
                                                                          (d.quant && d.D == 128 && d.live_splits <= 2))))
                  ? 1 : 0;
  // without the tcgen05 grid the streaming kernel also takes the single-segment codes parts
  d.scodes = (d.fstream && d.quant && d.D == 128 && !tc_launch) ? 1 : 0;
  const bool full = tc_launch && big_launch;   // persistent grids fill the GPU: fork side work after them
  // cut mode: each split's codes entries and FP16 entries are separate parts (one geometry for every
  // K2 kernel): codes parts go to the tcgen05 grid / the general kernel, FP16 parts to the stream
  d.cut_nq = (d.quant && ((kTcEnabled && d.D == 128 && d.use_tc) || d.fstream)) ? 1 : 0;
  static const bool no_absorb = getenv("CKV_ABSORB") && atoi(getenv("CKV_ABSORB")) == 0;
  d.absorb = (d.D >= 64 && !no_absorb) ? 1 : 0;   // k2_attend_split (D < 64) keeps plain 512-entry splits
  g_k2_launches = 0;
  cudaError_t e = cudaErrorInvalidValue;
  if (mid && !full && (e = cudaEventRecord(mid, s)) != cudaSuccess) return e;
  switch (d.D) {
    case 16: e = dispatch_g<16>(d, maps, c0, ccount, q, s); break;
    case 32: e = dispatch_g<32>(d, maps, c0, ccount, q, s); break;
    case 64: e = dispatch_g<64>(d, maps, c0, ccount, q, s); break;
    case 128: e = dispatch_g<128>(d, maps, c0, ccount, q, s); break;
  }
  if (e != cudaSuccess) return e;
  // the attention grids are submitted: a caller's side-stream work forked here (K1) runs beside
  // the combine instead of taking SM room from them (done before the grids when they cannot fill
  // the GPU -- no big tcgen05 launch -- so the side work overlaps them as before)
  if (mid && full && (e = cudaEventRecord(mid, s)) != cudaSuccess) return e;
  // K1 inline: the tcgen05 grid's programmatic dependent (its CTAs take the SM room the grid's
  // retiring CTAs leave), the combine its dependent in turn (waits for it, hence for the grid)
  const bool k1_inline = k1 && full && !mid;
  if (k1) k1->inlined = k1_inline ? 1 : 0;
  if (k1_inline) {
    if ((e = launch_confidence(d, *k1->c, k1->logits, k1->dtype, k1->ld, s, 0, nullptr, true)) != cudaSuccess) return e;
    ++g_k2_launches;
  }
  const size_t smem = (size_t)(3 * d.Hq + d.Hq * d.npart) * sizeof(float);
  const int live = std::min(d.cap, d.live_splits * kSplitTokens);   // entries any cache can hold now
  const int n4 = (live + 4 * kCombThreads - 1) / (4 * kCombThreads);
  const bool big = n4 * ccount >= 4 * 148;
  const int comb = d.comb_force >= 0 ? d.comb_force : (big ? 2 : 0);
  cudaLaunchAttribute pdl_attr[1];
  pdl_attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl_attr[0].val.programmaticStreamSerializationAllowed = 1;
  auto cfgc = [&](dim3 g, size_t sm) {   // the combine: K1's programmatic dependent when K1 is inline
    cudaLaunchConfig_t k = {};
    k.gridDim = g;
    k.blockDim = dim3(kCombThreads);
    k.dynamicSmemBytes = sm;
    k.stream = s;
    k.attrs = pdl_attr;
    k.numAttrs = k1_inline ? 1 : 0;
    return k;
  };
  if (comb == 2) {
    const size_t smem_st = kCombRing + 16 + smem;
    static size_t configured = 0;
    if (smem_st > configured) {
      cudaError_t ea = cudaFuncSetAttribute(k2_combine_staged<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_st);
      if (ea == cudaSuccess)
        ea = cudaFuncSetAttribute(k2_combine_staged<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_st);
      if (ea != cudaSuccess) return ea;
      configured = smem_st;
    }
    cudaLaunchConfig_t k = cfgc(dim3(n4, ccount), smem_st);
    e = wdump ? cudaLaunchKernelEx(&k, k2_combine_staged<true>, d, c0, out, wdump, (int)d.D)
              : cudaLaunchKernelEx(&k, k2_combine_staged<false>, d, c0, out, wdump, (int)d.D);
  } else if (comb == 1) {
    cudaLaunchConfig_t k = cfgc(dim3(n4, ccount), smem);
    e = wdump ? cudaLaunchKernelEx(&k, k2_combine<4, true>, d, c0, out, wdump, (int)d.D)
              : cudaLaunchKernelEx(&k, k2_combine<4, false>, d, c0, out, wdump, (int)d.D);
  } else {
    const int n1 = (live + kCombThreads - 1) / kCombThreads;
    cudaLaunchConfig_t k = cfgc(dim3(n1, ccount), smem);
    e = wdump ? cudaLaunchKernelEx(&k, k2_combine<1, true>, d, c0, out, wdump, (int)d.D)
              : cudaLaunchKernelEx(&k, k2_combine<1, false>, d, c0, out, wdump, (int)d.D);
  }
  if (e != cudaSuccess) return e;
  ++g_k2_launches;   // the combine
  return cudaGetLastError();
}

cudaError_t launch_stage_weights(const Dev& d, int c0, int ccount, const float* w, int shards, cudaStream_t s) {
  k2_stage_weights<<<dim3((d.cap + 255) / 256, ccount), 256, 0, s>>>(d, c0, ccount, w, shards);
  return cudaGetLastError();
}

cudaError_t launch_head_partial(const Dev& d, int c0, int ccount, const float* w, const double* acc_in, double* acc_out,
                                cudaStream_t s) {
  k2_head_partial<<<dim3((d.cap + 255) / 256, ccount), 256, 0, s>>>(d, c0, w, acc_in, acc_out);
  return cudaGetLastError();
}

cudaError_t launch_stage_mass(const Dev& d, int c0, int ccount, const double* acc, int total_heads, cudaStream_t s) {
  k2_stage_mass<<<dim3((d.cap + 255) / 256, ccount), 256, 0, s>>>(d, c0, acc, total_heads);
  return cudaGetLastError();
}

cudaError_t launch_stage_rows(const Dev& d, int layer, const double* rows, int ld, cudaStream_t s) {
  k2_stage_rows<<<dim3((d.cap + 255) / 256, d.B), 256, 0, s>>>(d, layer, rows, ld);
  return cudaGetLastError();
}

}  // namespace ckv

#ifdef CKV_TRACE
extern "C" int ckv_debug_ptrace(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(ckv::g_ptrace) ? bytes : sizeof(ckv::g_ptrace);
  return (int)cudaMemcpyFromSymbol(host, ckv::g_ptrace, n);
}
extern "C" int ckv_debug_timeline(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(ckv::g_tl) ? bytes : sizeof(ckv::g_tl);
  return (int)cudaMemcpyFromSymbol(host, ckv::g_tl, n);
}
extern "C" int ckv_debug_trace(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(ckv::g_trace) ? bytes : sizeof(ckv::g_trace);
  return (int)cudaMemcpyFromSymbol(host, ckv::g_trace, n);
}
#endif
