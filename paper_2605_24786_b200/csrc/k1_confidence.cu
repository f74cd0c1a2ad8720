// K1 — vocab-wide confidence in one pass over the logits.
//
// Replaces DecodePolicy._distribution + stable_softmax + confidence_score +
// select_budget + greedy _sample (policy.py:175-185, confidence.py:31-87).
// The distribution p is never materialised: each block reads its logits once
// (16-byte vectors), takes the block max m, then Z = sum e^(x-m),
// S = sum (x-m) e^(x-m), the top-2 logits and the arg-max index, all in fp64
// so the composite c matches the reference's fp64 NumPy to ~1e-15 and the
// tier decision c >= tau agrees except on exact ties. Partials are summed
// warp -> block; the last block of a sequence (ticket counter) merges
// the per-block partials (warp 0: strided lanes + a fixed shuffle tree, deterministic) and emits
//   H = ln Z - S/Z, H_norm = H / ln V, p1 = 1/Z, p2 = e^(l2-m)/Z,
//   margin = max(ln p1 - ln max(p2, 1e-12), 0), c = wH(1-H_norm)+wM sig(m)+wP p1.
// HBM traffic: exactly B * V * sizeof(logit) bytes read.
#include <cuda_bf16.h>

#include "ckv_internal.cuh"

namespace ckv {
namespace {

#ifdef CKV_TRACE
// per-CTA start / end (tools/trace_timeline.py)
constexpr int kK1TraceCtas = 8192;
__device__ unsigned long long g_k1trace[kK1TraceCtas][2];
__device__ __forceinline__ void k1stamp(int i) {
  const unsigned b = blockIdx.x + gridDim.x * blockIdx.y;
  if (threadIdx.x == 0 && b < kK1TraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k1trace[b][i] = t;
  }
}
#define K1_STAMP(i) k1stamp(i)
#else
#define K1_STAMP(i)
#endif

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

template <int DT>
__device__ __forceinline__ double load_logit(const void* base, int64_t i) {
  if (DT == CKV_DTYPE_F32) return (double)__ldg(reinterpret_cast<const float*>(base) + i);
  if (DT == CKV_DTYPE_F64) return __ldg(reinterpret_cast<const double*>(base) + i);
  return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
}

__device__ void finalize_impl(Dev& d, const Cfg& c, const Acc& r, int64_t V, int b);

// Called once per CTA by its last thread to finish: the grid's last CTA waits for the
// programmatic prerequisite grid (the tcgen05 grid, when K1 runs inline beside it), so this
// grid's completion implies that grid's while every other CTA exits at once (a wait in every CTA
// held K1's first wave on the SMs and kept its second wave off them until the grid's end).
__device__ __forceinline__ void k1_exit(const Dev& d) {
  __threadfence();
  if (atomicAdd(d.k1exit, 1) == (int)(gridDim.x * gridDim.y) - 1) {
    *d.k1exit = 0;
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
}
__device__ __forceinline__ void finalize(Dev d, const Cfg& c, const Acc& r, int64_t V, int b) {
  finalize_impl(d, c, r, V, b);
}

// Top-2 / arg-max part of acc_merge (disjoint index sets; ties keep the smaller index).
__device__ __forceinline__ void top_merge(Acc& a, double v1, double v2, int i1) {
  if (a.v1 > v1) {
    a.v2 = fmax(a.v2, v1);
  } else if (v1 > a.v1) {
    a.v2 = fmax(a.v1, v2); a.v1 = v1; a.i1 = i1;
  } else {   // equal top logits: duplicate maximum -> p2 == p1
    a.v2 = a.v1; a.i1 = min(a.i1, i1);
  }
}

// One block = kConfPerBlock consecutive logits of one sequence (kConfIters 16-byte vectors per
// thread, all loads issued up front). The block's max is found first (exact max of the inputs),
// so every exponential is taken against the same reference point: each element costs one
// independent fp64 exp, and the warp / block combination of (Z, S) is plain fp64 addition --
// no rescaling exp on the merge tree's critical path. Block partials (m, Z, S, top-2, arg-max)
// are merged by the sequence's last block against the global max (one exp per partial).
template <int DT, bool VEC>
__global__ void __launch_bounds__(kConfThreads)
k1_confidence(Dev d, Cfg c, const void* __restrict__ logits, int64_t ld, int nblk, int voff,
              double* __restrict__ partial_out) {
  constexpr int NE = kConfVec * kConfIters;   // elements per thread
  K1_STAMP(0);
  // inline in a step (a programmatic dependent of the tcgen05 grid): let the combine's CTAs be
  // placed as ours retire; every exit waits for the prerequisite grid so this grid's completion
  // implies it (no-ops when launched normally)
  asm volatile("griddepcontrol.launch_dependents;");
  const int b = blockIdx.y;
  const int blk = blockIdx.x;
  const int V = d.V;
  const char* row = reinterpret_cast<const char*>(logits) +
                    (size_t)b * ld * (DT == CKV_DTYPE_F64 ? 8 : DT == CKV_DTYPE_F32 ? 4 : 2);
  const bool temp = c.temp_mode != 0;
  const double T = c.temperature;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk0 = (int64_t)blk * kConfPerBlock;

  // ---- loads: vector it of this thread covers [i0(it), i0(it) + kConfVec) ----
  double x[NE];
  int nval[kConfIters];
#pragma unroll
  for (int it = 0; it < kConfIters; ++it) {
    const int64_t i0 = blk0 + ((int64_t)it * kConfThreads + threadIdx.x) * kConfVec;
    const int64_t left = (int64_t)V - i0;
    const int valid = left <= 0 ? 0 : left < kConfVec ? (int)left : kConfVec;
    nval[it] = valid;
    if (VEC && DT == CKV_DTYPE_F32 && valid == kConfVec) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(row) + i0 / 4);
      x[it * kConfVec + 0] = f.x; x[it * kConfVec + 1] = f.y; x[it * kConfVec + 2] = f.z; x[it * kConfVec + 3] = f.w;
    } else if (VEC && DT == CKV_DTYPE_F64 && valid == kConfVec) {
      const double2 f0 = __ldg(reinterpret_cast<const double2*>(row) + i0 / 2);
      const double2 f1 = __ldg(reinterpret_cast<const double2*>(row) + i0 / 2 + 1);
      x[it * kConfVec + 0] = f0.x; x[it * kConfVec + 1] = f0.y; x[it * kConfVec + 2] = f1.x; x[it * kConfVec + 3] = f1.y;
    } else {
#pragma unroll
      for (int j = 0; j < kConfVec; ++j) x[it * kConfVec + j] = j < valid ? load_logit<DT>(row, i0 + j) : 0.0;
    }
  }
  // ---- non-finite check, temperature (policy.py:178, fp64), thread max + top-2 in index order ----
  Acc a;
  acc_init(a);
#pragma unroll
  for (int it = 0; it < kConfIters; ++it) {
    const int i0 = (int)(blk0 + ((int64_t)it * kConfThreads + threadIdx.x) * kConfVec) + voff;
#pragma unroll
    for (int j = 0; j < kConfVec; ++j) {
      if (j >= nval[it]) continue;
      double& v = x[it * kConfVec + j];
      if (!isfinite(v)) { a.bad = 1; v = 0.0; }
      if (temp) v = v / T;
      a.m = fmax(a.m, v);
      if (v > a.v1) { a.v2 = a.v1; a.v1 = v; a.i1 = i0 + j; }
      else if (v == a.v1) { a.v2 = v; }
      else if (v > a.v2) { a.v2 = v; }
    }
  }
  // ---- block max ----
  __shared__ double s_m[kConfThreads / 32];
  __shared__ Acc wacc[kConfThreads / 32];
  __shared__ int s_last;
  double m = a.m;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) s_m[warp] = m;
  __syncthreads();
  double M = s_m[0];
#pragma unroll
  for (int w = 1; w < kConfThreads / 32; ++w) M = fmax(M, s_m[w]);
  // ---- Z, S against the block max: independent exps, plain sums ----
  double z = 0.0, sm = 0.0;
  if (M > -INFINITY) {
#pragma unroll
    for (int it = 0; it < kConfIters; ++it)
#pragma unroll
      for (int j = 0; j < kConfVec; ++j) {
        if (j >= nval[it]) continue;
        const double dd = x[it * kConfVec + j] - M;
        const double e = exp(dd);
        z += e;
        sm += dd * e;
      }
  }
  // warp: sums and top-2 (lane order: lower lanes hold lower indices)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    z += __shfl_down_sync(0xffffffffu, z, off);
    sm += __shfl_down_sync(0xffffffffu, sm, off);
    const double v1 = __shfl_down_sync(0xffffffffu, a.v1, off), v2 = __shfl_down_sync(0xffffffffu, a.v2, off);
    const int i1 = __shfl_down_sync(0xffffffffu, a.i1, off), bad = __shfl_down_sync(0xffffffffu, a.bad, off);
    top_merge(a, v1, v2, i1);
    a.bad |= bad;
  }
  if (lane == 0) {
    a.m = M; a.z = z; a.s = sm;
    wacc[warp] = a;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = wacc[0];
    for (int w = 1; w < kConfThreads / 32; ++w) {
      t.z += wacc[w].z;
      t.s += wacc[w].s;
      top_merge(t, wacc[w].v1, wacc[w].v2, wacc[w].i1);
      t.bad |= wacc[w].bad;
    }
    double* p = d.cpart + ((size_t)b * nblk + blk) * 8;
    p[0] = t.m; p[1] = t.z; p[2] = t.s; p[3] = t.v1; p[4] = t.v2;
    p[5] = (double)t.i1; p[6] = (double)t.bad;
    __threadfence();
    s_last = atomicAdd(&d.ticket[b], 1) == nblk - 1;
  }
  __syncthreads();
  if (!s_last || warp != 0) {
    K1_STAMP(1);
    if (threadIdx.x == 0 && !s_last) k1_exit(d);
    return;
  }
  // last block of the sequence: warp 0 merges the nblk block partials against their common max
  // (lane l holds blocks l, l + 32, ...; a fixed shuffle tree: deterministic)
  __threadfence();
  double gm = -INFINITY;
  for (int k = lane; k < nblk; k += 32) gm = fmax(gm, ((const volatile double*)d.cpart)[((size_t)b * nblk + k) * 8]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, off));
  Acc r;
  acc_init(r);
  double rz = 0.0, rs = 0.0;
  for (int k = lane; k < nblk; k += 32) {
    const volatile double* qp = d.cpart + ((size_t)b * nblk + k) * 8;
    const double bm = qp[0], bz = qp[1], bs = qp[2];
    if (bz > 0.0) {
      const double f = exp(bm - gm);
      rz += bz * f;
      rs += f * (bs + (bm - gm) * bz);
    }
    top_merge(r, qp[3], qp[4], (int)qp[5]);
    r.bad |= (int)qp[6];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    rz += __shfl_down_sync(0xffffffffu, rz, off);
    rs += __shfl_down_sync(0xffffffffu, rs, off);
    const double v1 = __shfl_down_sync(0xffffffffu, r.v1, off), v2 = __shfl_down_sync(0xffffffffu, r.v2, off);
    const int i1 = __shfl_down_sync(0xffffffffu, r.i1, off), bad = __shfl_down_sync(0xffffffffu, r.bad, off);
    top_merge(r, v1, v2, i1);
    r.bad |= bad;
  }
  K1_STAMP(1);
  if (lane != 0) return;
  r.m = gm; r.z = rz; r.s = rs;
  d.ticket[b] = 0;
  if (partial_out) {   // vocab-sharded mode: export this shard's merged tuple
    double* o = partial_out + (size_t)b * 8;
    o[0] = r.m; o[1] = r.z; o[2] = r.s; o[3] = r.v1; o[4] = r.v2; o[5] = (double)r.i1; o[6] = (double)r.bad;
    o[7] = 0.0;
    k1_exit(d);
    return;
  }
  finalize(d, c, r, V, b);
  k1_exit(d);
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
                              cudaStream_t s, int voff, double* partial_out, bool pdl) {
  const int nblk = (d.V + kConfPerBlock - 1) / kConfPerBlock;
  const bool vec = (reinterpret_cast<uintptr_t>(logits) % 16 == 0) && (ld % 4 == 0);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk, d.B);
  cfg.blockDim = dim3(kConfThreads);
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (dtype == CKV_DTYPE_F32)
    return vec ? cudaLaunchKernelEx(&cfg, k1_confidence<CKV_DTYPE_F32, true>, d, c, logits, ld, nblk, voff, partial_out)
               : cudaLaunchKernelEx(&cfg, k1_confidence<CKV_DTYPE_F32, false>, d, c, logits, ld, nblk, voff, partial_out);
  if (dtype == CKV_DTYPE_F64)   // the reference's own logits dtype (float64 NumPy rows, confidence.py:31-39)
    return vec ? cudaLaunchKernelEx(&cfg, k1_confidence<CKV_DTYPE_F64, true>, d, c, logits, ld, nblk, voff, partial_out)
               : cudaLaunchKernelEx(&cfg, k1_confidence<CKV_DTYPE_F64, false>, d, c, logits, ld, nblk, voff, partial_out);
  return cudaLaunchKernelEx(&cfg, k1_confidence<CKV_DTYPE_BF16, false>, d, c, logits, ld, nblk, voff, partial_out);
}

cudaError_t launch_confidence_merge(const Dev& d, const Cfg& c, const double* parts, int shards, int64_t vtotal,
                                    cudaStream_t s) {
  k1_merge<<<(d.B + 127) / 128, 128, 0, s>>>(d, c, parts, shards, vtotal);
  return cudaGetLastError();
}

}  // namespace ckv

#ifdef CKV_TRACE
extern "C" int ckv_debug_k1trace(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(ckv::g_k1trace) ? bytes : sizeof(ckv::g_k1trace);
  return (int)cudaMemcpyFromSymbol(host, ckv::g_k1trace, n);
}
#endif
