// K1 — vocab-wide confidence in one pass over the logits.
//
// Replaces DecodePolicy._distribution + stable_softmax + confidence_score +
// select_budget + greedy _sample (policy.py:175-185, confidence.py:31-87).
// The distribution p is never materialised: each thread streams 16-byte
// vectors of logits and keeps an online (max m, Z = sum e^(x-m),
// S = sum (x-m) e^(x-m)) plus the top-2 logits and the arg-max index, all in
// fp64 so the composite c matches the reference's fp64 NumPy to ~1e-15 and
// the tier decision c >= tau agrees except on exact ties. Partials are merged
// warp -> block -> grid; the last block of a sequence (ticket counter) merges
// the per-block partials (warp 0: strided lanes + a fixed shuffle tree, deterministic) and emits
//   H = ln Z - S/Z, H_norm = H / ln V, p1 = 1/Z, p2 = e^(l2-m)/Z,
//   margin = max(ln p1 - ln max(p2, 1e-12), 0), c = wH(1-H_norm)+wM sig(m)+wP p1.
// HBM traffic: exactly B * V * sizeof(logit) bytes read.
#include <cuda_bf16.h>

#include "ckv_internal.cuh"

namespace ckv {
namespace {

struct Acc {
  double m, z, s;   // online softmax moments (relative to m)
  double v1, v2;    // top-2 logits (multiset)
  int i1;           // arg-max (smallest index on ties)
  int bad;          // saw a non-finite logit
};

__device__ __forceinline__ void acc_init(Acc& a) {
  a.m = -INFINITY; a.z = 0.0; a.s = 0.0; a.v1 = -INFINITY; a.v2 = -INFINITY; a.i1 = 0x7fffffff; a.bad = 0;
}

// Merge b into a. Index sets are disjoint; ties on v1 keep the smaller index.
__device__ __forceinline__ void acc_merge(Acc& a, const Acc& b) {
  double M = fmax(a.m, b.m);
  double z = 0.0, s = 0.0;
  if (a.z > 0.0) { double f = exp(a.m - M); z += a.z * f; s += f * (a.s + (a.m - M) * a.z); }
  if (b.z > 0.0) { double f = exp(b.m - M); z += b.z * f; s += f * (b.s + (b.m - M) * b.z); }
  a.m = M; a.z = z; a.s = s;
  if (a.v1 > b.v1) {
    a.v2 = fmax(a.v2, b.v1);
  } else if (b.v1 > a.v1) {
    a.v2 = fmax(a.v1, b.v2); a.v1 = b.v1; a.i1 = b.i1;
  } else {  // equal top logits: duplicate maximum -> p2 == p1
    a.v2 = a.v1; a.i1 = min(a.i1, b.i1);
  }
  a.bad |= b.bad;
}

// Sequential update for a small group of consecutive elements (indices ascending).
template <int N>
__device__ __forceinline__ void acc_push(Acc& a, const double (&x)[N], int idx0, int valid) {
  double cmax = -INFINITY;
#pragma unroll
  for (int j = 0; j < N; ++j)
    if (j < valid) cmax = fmax(cmax, x[j]);
  if (cmax > a.m) {
    if (a.z > 0.0) {
      double f = exp(a.m - cmax);
      a.s = f * (a.s + (a.m - cmax) * a.z);
      a.z *= f;
    }
    a.m = cmax;
  }
#pragma unroll
  for (int j = 0; j < N; ++j) {
    if (j >= valid) break;
    double d = x[j] - a.m;
    double e = exp(d);
    a.z += e;
    a.s += d * e;
    if (x[j] > a.v1) { a.v2 = a.v1; a.v1 = x[j]; a.i1 = idx0 + j; }
    else if (x[j] == a.v1) { a.v2 = x[j]; }
    else if (x[j] > a.v2) { a.v2 = x[j]; }
  }
}

__device__ __forceinline__ Acc acc_shfl_down(const Acc& a, int off) {
  Acc b;
  b.m = __shfl_down_sync(0xffffffffu, a.m, off);
  b.z = __shfl_down_sync(0xffffffffu, a.z, off);
  b.s = __shfl_down_sync(0xffffffffu, a.s, off);
  b.v1 = __shfl_down_sync(0xffffffffu, a.v1, off);
  b.v2 = __shfl_down_sync(0xffffffffu, a.v2, off);
  b.i1 = __shfl_down_sync(0xffffffffu, a.i1, off);
  b.bad = __shfl_down_sync(0xffffffffu, a.bad, off);
  return b;
}

template <int DT>
__device__ __forceinline__ double load_logit(const void* base, int64_t i) {
  if (DT == CKV_DTYPE_F32) return (double)__ldg(reinterpret_cast<const float*>(base) + i);
  if (DT == CKV_DTYPE_F64) return __ldg(reinterpret_cast<const double*>(base) + i);
  return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
}

__device__ void finalize_impl(Dev& d, const Cfg& c, const Acc& r, int64_t V, int b);
__device__ __forceinline__ void finalize(Dev d, const Cfg& c, const Acc& r, int64_t V, int b) {
  finalize_impl(d, c, r, V, b);
}

template <int DT, bool VEC>
__global__ void __launch_bounds__(kConfThreads)
k1_confidence(Dev d, Cfg c, const void* __restrict__ logits, int64_t ld, int nblk, int voff,
              double* __restrict__ partial_out) {
  const int b = blockIdx.y;
  const int blk = blockIdx.x;
  const int V = d.V;
  const char* row = reinterpret_cast<const char*>(logits) +
                    (size_t)b * ld * (DT == CKV_DTYPE_F64 ? 8 : DT == CKV_DTYPE_F32 ? 4 : 2);
  const bool temp = c.temp_mode != 0;
  const double T = c.temperature;

  Acc a;
  acc_init(a);
  const int64_t blk0 = (int64_t)blk * kConfPerBlock;
#pragma unroll 1
  for (int it = 0; it < kConfIters; ++it) {
    const int64_t i0 = blk0 + ((int64_t)it * kConfThreads + threadIdx.x) * kConfVec;
    if (i0 >= V) break;
    double x[kConfVec];
    const int64_t left = (int64_t)V - i0;
    int valid = left < kConfVec ? (int)left : kConfVec;
    if (VEC && DT == CKV_DTYPE_F32 && valid == kConfVec) {
      float4 f = __ldg(reinterpret_cast<const float4*>(row) + i0 / 4);
      x[0] = f.x; x[1] = f.y; x[2] = f.z; x[3] = f.w;
    } else if (VEC && DT == CKV_DTYPE_F64 && valid == kConfVec) {
      const double2 f0 = __ldg(reinterpret_cast<const double2*>(row) + i0 / 2);
      const double2 f1 = __ldg(reinterpret_cast<const double2*>(row) + i0 / 2 + 1);
      x[0] = f0.x; x[1] = f0.y; x[2] = f1.x; x[3] = f1.y;
    } else {
#pragma unroll
      for (int j = 0; j < kConfVec; ++j) x[j] = j < valid ? load_logit<DT>(row, i0 + j) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < kConfVec; ++j) {
      if (j < valid) {
        if (!isfinite(x[j])) { a.bad = 1; x[j] = 0.0; }
        if (temp) x[j] = x[j] / T;   // policy.py:178: logits / temperature in fp64
      }
    }
    acc_push<kConfVec>(a, x, (int)i0 + voff, valid);
  }

  // warp -> block
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Acc o = acc_shfl_down(a, off);
    acc_merge(a, o);   // lane order: lower lanes hold lower indices
  }
  __shared__ Acc wacc[kConfThreads / 32];
  __shared__ int s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) wacc[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = wacc[0];
    for (int w = 1; w < kConfThreads / 32; ++w) acc_merge(t, wacc[w]);
    double* p = d.cpart + ((size_t)b * nblk + blk) * 8;
    p[0] = t.m; p[1] = t.z; p[2] = t.s; p[3] = t.v1; p[4] = t.v2;
    p[5] = (double)t.i1; p[6] = (double)t.bad;
    __threadfence();
    s_last = atomicAdd(&d.ticket[b], 1) == nblk - 1;
  }
  __syncthreads();
  if (!s_last || warp != 0) return;
  // last block of the sequence: warp 0 merges the nblk block partials, lane l the blocks
  // l, l + 32, ... in order, then a fixed shuffle tree (deterministic)
  __threadfence();
  Acc r;
  acc_init(r);
  for (int k = lane; k < nblk; k += 32) {
    const volatile double* q = d.cpart + ((size_t)b * nblk + k) * 8;
    Acc u;
    u.m = q[0]; u.z = q[1]; u.s = q[2]; u.v1 = q[3]; u.v2 = q[4];
    u.i1 = (int)q[5]; u.bad = (int)q[6];
    acc_merge(r, u);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Acc o = acc_shfl_down(r, off);
    acc_merge(r, o);
  }
  if (lane != 0) return;
  d.ticket[b] = 0;
  if (partial_out) {   // vocab-sharded mode: export this shard's merged tuple
    double* o = partial_out + (size_t)b * 8;
    o[0] = r.m; o[1] = r.z; o[2] = r.s; o[3] = r.v1; o[4] = r.v2; o[5] = (double)r.i1; o[6] = (double)r.bad;
    o[7] = 0.0;
    return;
  }
  finalize(d, c, r, V, b);
}

// Rank-order merge of vocab-shard tuples ([shards][B][8]) and the final features.
__global__ void k1_merge(Dev d, Cfg c, const double* __restrict__ parts, int shards, int64_t vtotal) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= d.B) return;
  Acc r;
  acc_init(r);
  for (int k = 0; k < shards; ++k) {
    const double* q = parts + ((size_t)k * d.B + b) * 8;
    Acc u;
    u.m = q[0]; u.z = q[1]; u.s = q[2]; u.v1 = q[3]; u.v2 = q[4]; u.i1 = (int)q[5]; u.bad = (int)q[6];
    acc_merge(r, u);
  }
  finalize(d, c, r, vtotal, b);
}

// Features from the merged moments (confidence.py:64-75): H = ln Z - S/Z, H_norm = H/ln V,
// p1 = 1/Z, p2 = e^(l2-m)/Z floored at 1e-12, margin = max(ln p1 - ln p2, 0).
__device__ void finalize_impl(Dev& d, const Cfg& c, const Acc& r, int64_t V, int b) {
  const double Z = r.z;
  const double H = log(Z) - r.s / Z;
  const double hn = H / log((double)V);
  const double p1 = 1.0 / Z;                     // e^(v1 - m) = 1
  const double p2 = fmax(exp(r.v2 - r.m) / Z, 1e-12);
  const double margin = fmax(log(p1) - log(p2), 0.0);
  const double sig = 1.0 / (1.0 + exp(-margin));
  const double score = c.wH * (1.0 - hn) + c.wM * sig + c.wP * p1;
  ckv_seq_record out;
  out.score = score; out.entropy_norm = hn; out.margin = margin; out.margin_sig = sig;
  out.top_prob = p1;
  out.tier_high = score >= c.tau ? 1 : 0;        // confidence.py:85-87
  out.token = c.temp_mode ? -1 : r.i1;           // greedy argmax, ties -> smallest id
  out.status = r.bad ? kStNonFinite : 0;
  out.pad = 0;
  d.conf[b] = out;
}

}  // namespace

cudaError_t launch_confidence(const Dev& d, const Cfg& c, const void* logits, int dtype, int64_t ld,
                              cudaStream_t s, int voff, double* partial_out) {
  const int nblk = (d.V + kConfPerBlock - 1) / kConfPerBlock;
  dim3 grid(nblk, d.B);
  const bool vec = (reinterpret_cast<uintptr_t>(logits) % 16 == 0) && (ld % 4 == 0);
  if (dtype == CKV_DTYPE_F32) {
    if (vec) k1_confidence<CKV_DTYPE_F32, true><<<grid, kConfThreads, 0, s>>>(d, c, logits, ld, nblk, voff, partial_out);
    else k1_confidence<CKV_DTYPE_F32, false><<<grid, kConfThreads, 0, s>>>(d, c, logits, ld, nblk, voff, partial_out);
  } else if (dtype == CKV_DTYPE_F64) {
    // the reference's own logits dtype (float64 NumPy rows, confidence.py:31-39)
    if (vec) k1_confidence<CKV_DTYPE_F64, true><<<grid, kConfThreads, 0, s>>>(d, c, logits, ld, nblk, voff, partial_out);
    else k1_confidence<CKV_DTYPE_F64, false><<<grid, kConfThreads, 0, s>>>(d, c, logits, ld, nblk, voff, partial_out);
  } else {
    k1_confidence<CKV_DTYPE_BF16, false><<<grid, kConfThreads, 0, s>>>(d, c, logits, ld, nblk, voff, partial_out);
  }
  return cudaGetLastError();
}

cudaError_t launch_confidence_merge(const Dev& d, const Cfg& c, const double* parts, int shards, int64_t vtotal,
                                    cudaStream_t s) {
  k1_merge<<<(d.B + 127) / 128, 128, 0, s>>>(d, c, parts, shards, vtotal);
  return cudaGetLastError();
}

}  // namespace ckv
