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
#include "ckv_internal.cuh"

namespace ckv {
namespace {

constexpr int kConsumerWarps = 4;
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
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
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
  const int n8 = d.n8[c];
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
            const int r0 = (rbase + s_slot[j + g0]) * d.Hkv + h, r1 = (rbase + s_slot[j + g0 + 1]) * d.Hkv + h;
            const int r2 = (rbase + s_slot[j + g0 + 2]) * d.Hkv + h, r3 = (rbase + s_slot[j + g0 + 3]) * d.Hkv + h;
            if (g0 >= n8s) {
              tma_gather4(ko, &maps.kf, r0, r1, r2, r3, full);
              tma_gather4(vo, &maps.vf, r0, r1, r2, r3, full);
            } else {
              tma_gather4(ko, &maps.kq, r0, r1, r2, r3, full);
              tma_gather4(vo, &maps.vq, r0, r1, r2, r3, full);
            }
          } else {
            for (int r = g0; r < min(g0 + 4, nrow); ++r) {
              const size_t off = ((size_t)rbase + s_slot[j + r]) * row + (size_t)h * D;
              if (r < n8s) {
                tma_row(ko + (r - g0) * D, d.kq + off, D, full);
                tma_row(vo + (r - g0) * D, d.vq + off, D, full);
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
    float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.cap;

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
          if (i < end) scoreg[(size_t)g * d.cap + i] = sv;
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
    const size_t pbase = ((size_t)c * Hq + (size_t)h * G) * d.nsplit + split;
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
      const size_t pi = pbase + (size_t)g * d.nsplit;
      d.po[pi * D + dd] = O;
      if (dd == 0) { d.pm[pi] = M; d.pz[pi] = Z; }
    }
  }
}

// Combine split partials -> out; normalised weights -> head mean (fp64) -> abar.
__global__ void __launch_bounds__(256)
k2_combine(Dev d, int c0, float* __restrict__ out, float* __restrict__ wdump, int D) {
  extern __shared__ float sm[];
  const int Hq = d.Hq, nsp = d.nsplit;
  float* sM = sm;                 // [Hq]
  float* sZ = sM + Hq;            // [Hq]
  float* sF = sZ + Hq;            // [Hq][nsp] rescale factors
  const int c = c0 + blockIdx.y;
  const int n = d.len[c];
  const int nused = (n + kSplitTokens - 1) / kSplitTokens;
  for (int g = threadIdx.x; g < Hq; g += blockDim.x) {
    const size_t pi = ((size_t)c * Hq + g) * nsp;
    float M = -INFINITY;
    for (int s = 0; s < nused; ++s) M = fmaxf(M, d.pm[pi + s]);
    float Z = 0.f;
    for (int s = 0; s < nused; ++s) {
      const float f = (d.pm[pi + s] == -INFINITY) ? 0.f : expf(d.pm[pi + s] - M);
      sF[g * nsp + s] = f;
      Z += f * d.pz[pi + s];
    }
    sM[g] = M;
    sZ[g] = Z;
  }
  __syncthreads();
  if (blockIdx.x == 0) {
    if (out) {
      for (int idx = threadIdx.x; idx < Hq * D; idx += blockDim.x) {
        const int g = idx / D, dd = idx % D;
        const size_t pi = ((size_t)c * Hq + g) * nsp;
        float o = 0.f;
        for (int s = 0; s < nused; ++s) o += sF[g * nsp + s] * d.po[(pi + s) * D + dd];
        out[((size_t)(c - c0) * Hq + g) * D + dd] = sZ[g] > 0.f ? o / sZ[g] : 0.f;
      }
    }
    if (threadIdx.x == 0) d.att_len[c] = n;
  }
  const int per = (d.cap + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per, i1 = min(n, i0 + per);
  const double hq = (double)Hq;
  const float* sc = d.score + (size_t)c * Hq * d.cap;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double a = 0.0;
    for (int g = 0; g < Hq; ++g) {
      const float w = __fdiv_rn(expf(sc[(size_t)g * d.cap + i] - sM[g]), sZ[g]);
      if (wdump) wdump[((size_t)(c - c0) * Hq + g) * d.cap + i] = w;
      a = __dadd_rn(a, (double)w);
    }
    d.abar[(size_t)c * d.cap + i] = __ddiv_rn(a, hq);
  }
}

// Parity hook: head mean of host-supplied fp64 rows (update_attention_ema input).
__global__ void k2_stage_rows(Dev d, int layer, const double* __restrict__ rows, int ld) {
  const int b = blockIdx.y;
  const int c = layer * d.B + b;
  const int n = d.len[c];
  const int Hq = d.Hq;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int g = 0; g < Hq; ++g) a = __dadd_rn(a, rows[((size_t)b * Hq + g) * ld + i]);
    d.abar[(size_t)c * d.cap + i] = __ddiv_rn(a, (double)Hq);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) d.att_len[c] = n;
}

template <int D, int G>
cudaError_t launch_split(const Dev& d, const Maps& maps, int c0, int ccount, const __half* q, cudaStream_t s) {
  using T = Tr<D, G>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k2_attend_split<D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(d.nsplit, d.Hkv, ccount);
  k2_attend_split<D, G><<<grid, kThreads, T::SMEM, s>>>(d, maps, c0, q, (float)(1.0 / sqrt((double)D)));
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

bool attend_supported(int D, int G) {
  const bool dok = D == 16 || D == 32 || D == 64 || D == 128;
  const bool gok = G == 1 || G == 2 || G == 4 || G == 5 || G == 8;
  return dok && gok;
}

cudaError_t launch_attend(const Dev& d, const Maps& maps, int c0, int ccount, const __half* q,
                          float* out, float* wdump, cudaStream_t s) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (d.D) {
    case 16: e = dispatch_g<16>(d, maps, c0, ccount, q, s); break;
    case 32: e = dispatch_g<32>(d, maps, c0, ccount, q, s); break;
    case 64: e = dispatch_g<64>(d, maps, c0, ccount, q, s); break;
    case 128: e = dispatch_g<128>(d, maps, c0, ccount, q, s); break;
  }
  if (e != cudaSuccess) return e;
  const int nchunk = (d.cap + 1023) / 1024;
  const size_t smem = (size_t)(2 * d.Hq + d.Hq * d.nsplit) * sizeof(float);
  k2_combine<<<dim3(nchunk, ccount), 256, smem, s>>>(d, c0, out, wdump, d.D);
  return cudaGetLastError();
}

cudaError_t launch_stage_rows(const Dev& d, int layer, const double* rows, int ld, cudaStream_t s) {
  k2_stage_rows<<<dim3((d.cap + 255) / 256, d.B), 256, 0, s>>>(d, layer, rows, ld);
  return cudaGetLastError();
}

}  // namespace ckv
