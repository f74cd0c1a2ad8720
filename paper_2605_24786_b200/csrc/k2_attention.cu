// K2 — split-K online-softmax decode attention over the mixed FP16/INT8 cache,
// plus the combine / head-mean epilogue that stages the EMA input.
//
// Replaces tiled_attention (attention.py:60-102), LayerCache.read_block +
// dequantize (cache.py:238-252, quantizer.py:37-39) and the head-mean of
// update_attention_ema (cache.py:171). Grid = (split, kv head, cache): each CTA
// streams kSplitTokens tokens of one KV head and serves all G = Hq/Hkv query
// heads of the group from the same K/V bytes (GQA), so every K/V byte is read
// from HBM exactly once per step.
//
// Per warp-iteration a warp covers TT = RPW*U tokens: a token row (D dims of
// one KV head) is spread over LPR = D/8 lanes holding 8 dims each (one 16-byte
// fp16 vector, or 8 INT8 codes + their segment's fp32 scales). q.k partials
// for the U*G (token, head) pairs are reduced across the LPR lanes with a
// recursive-halving butterfly (log2(LPR)..U*G/LPR shuffles per pair, not
// U*G*log2(LPR)), the running max / rescale uses a warp-private smem tile, and
// P.V accumulates with packed fp32x2 FMA (FFMA2, sm_100). INT8 codes are
// widened with PRMT + FADD (exact) and dequantised code*scale in fp32 exactly
// as the reference does before use.
//
// Split partials (m, z, acc) go to scratch; k2_combine merges them (out) and
// turns the raw fp32 scores into the normalised weights the EMA consumes,
// summing heads sequentially in fp64 and dividing by Hq (cache.py:171's
// NumPy axis-0 mean) into abar[c][i].
#include "ckv_internal.cuh"

namespace ckv {
namespace {

constexpr int kAttnWarps = 4;

__host__ __device__ constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }
__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

template <int D, int G>
struct Tr {
  static constexpr int LPR = D / 8;                      // lanes per token row
  static constexpr int RPW = 32 / LPR;                   // rows per warp instruction
  static constexpr int U0 = D >= 64 ? 4 : (D == 32 ? 2 : 1);
  static constexpr int U = (G >= 5 && U0 > 1) ? U0 / 2 : U0;   // keep registers under the cap
  static constexpr int TT = RPW * U;                     // tokens per warp iteration
  static constexpr int K = U * G;                        // (token, head) dots per lane group
  static constexpr int KP = pow2ceil(K);
  static constexpr int HS = ilog2(cmin(KP, LPR));        // halving steps
  static constexpr int CNT = KP >= LPR ? KP / LPR : 1;   // values held per lane afterwards
  static constexpr int REP = KP >= LPR ? 1 : LPR / KP;   // lanes holding the same value
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

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

__device__ __forceinline__ void half8_to_f2(const uint4& w, float2 (&o)[4]) {
  o[0] = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
  o[1] = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
  o[2] = __half22float2(*reinterpret_cast<const __half2*>(&w.z));
  o[3] = __half22float2(*reinterpret_cast<const __half2*>(&w.w));
}

// 8 signed int8 codes -> 8 exact floats: bias to unsigned, splice into the
// mantissa of 2^23, subtract 2^23 + 128.
__device__ __forceinline__ void code8_to_f2(const uint2& w, float2 (&o)[4]) {
  const unsigned a = w.x ^ 0x80808080u, b = w.y ^ 0x80808080u;
  const float k = 8388736.0f;
  o[0] = make_float2(__int_as_float(__byte_perm(a, 0x4B000000u, 0x7440)) - k,
                     __int_as_float(__byte_perm(a, 0x4B000000u, 0x7441)) - k);
  o[1] = make_float2(__int_as_float(__byte_perm(a, 0x4B000000u, 0x7442)) - k,
                     __int_as_float(__byte_perm(a, 0x4B000000u, 0x7443)) - k);
  o[2] = make_float2(__int_as_float(__byte_perm(b, 0x4B000000u, 0x7440)) - k,
                     __int_as_float(__byte_perm(b, 0x4B000000u, 0x7441)) - k);
  o[3] = make_float2(__int_as_float(__byte_perm(b, 0x4B000000u, 0x7442)) - k,
                     __int_as_float(__byte_perm(b, 0x4B000000u, 0x7443)) - k);
}

__device__ __forceinline__ void dequant(float2 (&x)[4], const float* sc) {
  const float4 s0 = __ldg(reinterpret_cast<const float4*>(sc));
  const float4 s1 = __ldg(reinterpret_cast<const float4*>(sc) + 1);
  x[0] = fmul2(x[0], make_float2(s0.x, s0.y));
  x[1] = fmul2(x[1], make_float2(s0.z, s0.w));
  x[2] = fmul2(x[2], make_float2(s1.x, s1.y));
  x[3] = fmul2(x[3], make_float2(s1.z, s1.w));
}

template <int D, int G>
__global__ void __launch_bounds__(kAttnWarps * 32, 3)
k2_attend_split(Dev d, int c0, const __half* __restrict__ q, float qscale) {
  using T = Tr<D, G>;
  const int c = c0 + blockIdx.z;
  const int h = blockIdx.y;
  const int split = blockIdx.x;
  const int n = d.len[c];
  const int begin = split * kSplitTokens;
  if (begin >= n) return;
  const int end = min(n, begin + kSplitTokens);
  const int n8 = d.n8[c];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = lane / T::LPR, rl = lane % T::LPR;
  const int Hq = d.Hq;
  const size_t row = (size_t)d.Hkv * D;
  const size_t cbase = (size_t)c * d.cap;

  __shared__ __align__(16) float sS[kAttnWarps][G][T::TT];
  __shared__ __align__(16) float sP[kAttnWarps][G][T::TT];
  __shared__ float wm[kAttnWarps][G], wz[kAttnWarps][G];
  __shared__ float wacc[kAttnWarps][G][D];

  // q for the G heads of this KV head, pre-scaled by 1/sqrt(D)
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
  float* scoreg = d.score + ((size_t)c * Hq + (size_t)h * G) * d.cap;

#pragma unroll 1
  for (int tb = begin + warp * T::TT; tb < end; tb += kAttnWarps * T::TT) {
    // ---- load U token rows (K and V) per lane group ---------------------------------
    float2 kx[T::U][4], vx[T::U][4];
    bool ok[T::U];
#pragma unroll
    for (int u = 0; u < T::U; ++u) {
      const int i = tb + u * T::RPW + rg;
      ok[u] = i < end;
      if (ok[u]) {
        const int ps = __ldg(d.slot + cbase + i);
        const size_t off = ((size_t)c * d.cap + ps) * row + (size_t)h * D + rl * 8;
        if (i >= n8) {
          half8_to_f2(ldg_stream(d.kf + off), kx[u]);
          half8_to_f2(ldg_stream(d.vf + off), vx[u]);
        } else {
          const int sg = __ldg(d.seg + cbase + i);
          const size_t soff = (((size_t)c * d.smax + sg) * d.Hkv + h) * D + rl * 8;
          code8_to_f2(ldg_stream8(d.kq + off), kx[u]);
          code8_to_f2(ldg_stream8(d.vq + off), vx[u]);
          dequant(kx[u], d.ksc + soff);
          dequant(vx[u], d.vsc + soff);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) kx[u][j] = vx[u][j] = make_float2(0.f, 0.f);
      }
    }
    // ---- q.k partials over this lane's 8 dims ---------------------------------------
    float v[T::KP];
#pragma unroll
    for (int k = 0; k < T::KP; ++k) v[k] = 0.f;
#pragma unroll
    for (int u = 0; u < T::U; ++u) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float2 s2 = fmul2(qv[g][0], kx[u][0]);
#pragma unroll
        for (int j = 1; j < 4; ++j) s2 = ffma2(qv[g][j], kx[u][j], s2);
        v[u * G + g] = s2.x + s2.y;
      }
    }
    // ---- recursive-halving reduce across the LPR lanes of the row group -------------
#pragma unroll
    for (int s = 0, S = T::KP; s < T::HS; ++s, S >>= 1) {
      const int o = (T::LPR >> 1) >> s;
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
    // lane holds values [hb, hb + CNT) of the U*G (u, g) pairs
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
        sS[warp][g][t] = sv;
        if (i < end) scoreg[(size_t)g * d.cap + i] = sv;
      }
    }
    __syncwarp();
    // ---- tile max, rescale factors ---------------------------------------------------
    float corr[G], mn[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float tm = -INFINITY;
#pragma unroll
      for (int t = 0; t < T::TT; t += 4) {
        const float4 s4 = *reinterpret_cast<const float4*>(&sS[warp][g][t]);
        tm = fmaxf(tm, fmaxf(fmaxf(s4.x, s4.y), fmaxf(s4.z, s4.w)));
      }
      mn[g] = fmaxf(m[g], tm);
      corr[g] = (m[g] == mn[g]) ? 1.f : expf(m[g] - mn[g]);
      zp[g] *= corr[g];   // old partial sums move to the new max before this tile's p join
    }
    // ---- probabilities (computed once per (token, head) by its holder lane) --------
#pragma unroll
    for (int k = 0; k < T::CNT; ++k) {
      const int idx = hb + k;
      if (writer && idx < T::K) {
        const int u = idx / G, g = idx % G;
        const int t = u * T::RPW + rg;
        const float sv = sS[warp][g][t];
        const float p = (sv == -INFINITY) ? 0.f : expf(sv - mn[g]);
        sP[warp][g][t] = p;
        zp[g] += p;
      }
    }
    __syncwarp();
    // ---- P.V --------------------------------------------------------------------------
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
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float p = sP[warp][g][t];
        const float2 p2 = make_float2(p, p);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[g][j] = ffma2(p2, vx[u][j], acc[g][j]);
      }
    }
    __syncwarp();   // sS/sP are rewritten by the next iteration
  }

  // ---- reduce acc across row groups; z across the warp ---------------------------------
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

  if (lane < T::LPR) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wacc[warp][g][rl * 8 + 2 * j] = acc[g][j].x;
        wacc[warp][g][rl * 8 + 2 * j + 1] = acc[g][j].y;
      }
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) { wm[warp][g] = m[g]; wz[warp][g] = zp[g]; }
  }
  __syncthreads();
  const size_t pbase = ((size_t)c * Hq + (size_t)h * G) * d.nsplit + split;
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int g = idx / D, dd = idx % D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, wm[w][g]);
    float O = 0.f, Z = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      if (wm[w][g] == -INFINITY) continue;
      const float f = expf(wm[w][g] - M);
      O += f * wacc[w][g][dd];
      Z += f * wz[w][g];
    }
    const size_t pi = pbase + (size_t)g * d.nsplit;
    d.po[pi * D + dd] = O;
    if (dd == 0) { d.pm[pi] = M; d.pz[pi] = Z; }
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
  const double inv_h = (double)Hq;
  const float* sc = d.score + (size_t)c * Hq * d.cap;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    double a = 0.0;
    for (int g = 0; g < Hq; ++g) {
      const float w = __fdiv_rn(expf(sc[(size_t)g * d.cap + i] - sM[g]), sZ[g]);
      if (wdump) wdump[((size_t)(c - c0) * Hq + g) * d.cap + i] = w;
      a = __dadd_rn(a, (double)w);
    }
    d.abar[(size_t)c * d.cap + i] = __ddiv_rn(a, inv_h);
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
void launch_split(const Dev& d, int c0, int ccount, const __half* q, cudaStream_t s) {
  dim3 grid(d.nsplit, d.Hkv, ccount);
  k2_attend_split<D, G><<<grid, kAttnWarps * 32, 0, s>>>(d, c0, q, (float)(1.0 / sqrt((double)D)));
}

template <int D>
bool dispatch_g(const Dev& d, int c0, int ccount, const __half* q, cudaStream_t s) {
  switch (d.G) {
    case 1: launch_split<D, 1>(d, c0, ccount, q, s); return true;
    case 2: launch_split<D, 2>(d, c0, ccount, q, s); return true;
    case 4: launch_split<D, 4>(d, c0, ccount, q, s); return true;
    case 5: launch_split<D, 5>(d, c0, ccount, q, s); return true;
    case 8: launch_split<D, 8>(d, c0, ccount, q, s); return true;
    default: return false;
  }
}

}  // namespace

bool attend_supported(int D, int G) {
  const bool dok = D == 16 || D == 32 || D == 64 || D == 128;
  const bool gok = G == 1 || G == 2 || G == 4 || G == 5 || G == 8;
  return dok && gok;
}

cudaError_t launch_attend(const Dev& d, int c0, int ccount, const __half* q, float* out,
                          float* wdump, cudaStream_t s) {
  bool ok = false;
  switch (d.D) {
    case 16: ok = dispatch_g<16>(d, c0, ccount, q, s); break;
    case 32: ok = dispatch_g<32>(d, c0, ccount, q, s); break;
    case 64: ok = dispatch_g<64>(d, c0, ccount, q, s); break;
    case 128: ok = dispatch_g<128>(d, c0, ccount, q, s); break;
  }
  if (!ok) return cudaErrorInvalidValue;
  cudaError_t e = cudaGetLastError();
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
