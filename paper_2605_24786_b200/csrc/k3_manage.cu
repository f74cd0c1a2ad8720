// K3 — rank + select + compact (one CTA per (layer, sequence) cache) and
// K4 — INT8 demotion + append (one CTA per (KV head, cache)).
//
// K3 replaces ConfKVEngine._manage's per-layer body (policy.py:256-274):
// update_attention_ema's EMA commit (cache.py:172-177), layer_budget
// (policy.py:249-254), rank_candidates / select_victims / evict_to_budget
// (policy.py:72-127), LayerCache.compact + _drop_empty_segments
// (cache.py:181-234), the aged-set selection of apply_fp16_window
// (quantizer.py:42-64) and the metadata half of append (cache.py:111-132,
// policy.py:203-206).
//
// Exactness: the EMA and the composite are fp64 with every product and sum
// rounded separately (__dmul_rn/__dadd_rn, no FMA contraction), exactly as
// NumPy evaluates `lam*ema + (1-lam)*mean` and `alpha*a + (1-alpha)*r`.
// Composites are >= +0.0, so their IEEE bit patterns order as uint64 keys;
// victims are the `excess` smallest (key, index) pairs, found with an 8-pass
// 8-bit radix select plus an index-ordered scan over the threshold ties
// (np.lexsort((index, composite)) semantics), or a block arg-min when
// excess == 1 (the steady state).
//
// Storage moves are metadata only: K/V rows stay in their physical slots and
// the logical->physical `slot` map is compacted with the rest of the
// per-entry metadata (25 B/entry) in index order, chunk by chunk (dst <= src,
// all reads of a chunk complete before its writes). Victim slots return to a
// free stack; segments whose last member is evicted return to the segment
// pool (the reference's renumbering is a naming artifact; ckv_read_cache
// reports reference-numbered ids).
#include <algorithm>

#include "ckv_internal.cuh"

namespace ckv {
namespace {

constexpr int kTBig = kManageThreads;   // K3 block (512); 256 for many short caches (launch_manage)
constexpr int kU = 4;   // entries per thread per pass in the latency-bound streaming loops
// Staged fast path (composite keys, at most one victim, n <= kStage): every metadata array of
// the cache is read ONCE into shared memory (EMA committed on the way), min / max, keys and the
// arg-min run from shared memory, and the order-preserving shift is stored from it -- one
// global round trip for what took seven (EMA, min / max, keys, four shift chunks).
constexpr int kStage = 4352;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
constexpr int kStageBytes(int n) { return n * (8 + 4 * 4 + 1); }

// Debug build (-DCKV_TRACE): %globaltimer stamps at K3's phase boundaries per cache (block),
// read back with ckv_debug_k3trace() (tools/trace_k3.py).
#ifdef CKV_TRACE
constexpr int kK3TraceCaches = 4096;
__device__ unsigned long long g_k3trace[kK3TraceCaches][8];
__device__ __forceinline__ void k3stamp(int i) {
  if (threadIdx.x == 0 && blockIdx.x < kK3TraceCaches) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k3trace[blockIdx.x][i] = t;
  }
}
#define K3_STAMP(i) k3stamp(i)
// K4 per-CTA start / end (tools/trace_timeline.py)
constexpr int kK4TraceCtas = 8192;
__device__ unsigned long long g_k4trace[kK4TraceCtas][2];
__device__ __forceinline__ void k4stamp(int i) {
  const unsigned b = blockIdx.x + gridDim.x * blockIdx.y;
  if (threadIdx.x == 0 && b < kK4TraceCtas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k4trace[b][i] = t;
  }
}
#define K4_STAMP(i) k4stamp(i)
#else
#define K3_STAMP(i)
#define K4_STAMP(i)
#endif

// Exclusive block scan of a 0/1 flag. s_w must hold 33 ints.
__device__ __forceinline__ int block_scan(int flag, int* s_w, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, flag);
  const int wr = __popc(bal & ((1u << lane) - 1u));
  if (lane == 0) s_w[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const int v = lane < nw ? s_w[lane] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    s_w[lane] = x - v;
    if (lane == 31) s_w[32] = x;
  }
  __syncthreads();
  const int r = s_w[warp] + wr;
  total = s_w[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ int block_sum(int v, int* s_w) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < nw; ++w) s += s_w[w];
    s_w[32] = s;
  }
  __syncthreads();
  const int r = s_w[32];
  __syncthreads();
  return r;
}

// 8-pass 8-bit radix select of the `excess`-th smallest key among keys[base + 0 .. cut):
// s_T = the threshold key, s_need = how many keys equal to it are victims (lowest index
// first), s_vi = -1 (general victim set).
template <int kT>
__device__ __forceinline__ void radix_select(const Dev& d, size_t base, int cut, int excess, int* s_hist,
                                             int* s_red_i, unsigned long long& s_T, int& s_need, int& s_vi) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned long long prefix = 0, pmask = 0;
  int krem = excess;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int j = tid; j < 256; j += kT) s_hist[j] = 0;
    __syncthreads();
    for (int i = tid; i < cut; i += kT) {
      const unsigned long long key = d.keys[base + i];
      if ((key & pmask) == prefix) atomicAdd(&s_hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (warp == 0) {
      int hv[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { hv[j] = s_hist[lane * 8 + j]; sum += hv[j]; }
      int x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int before = x - sum;   // keys in bins < lane*8
      if (before < krem && krem <= x) {
        int acc = before;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (acc < krem && krem <= acc + hv[j]) { s_red_i[0] = lane * 8 + j; s_red_i[1] = acc; }
          acc += hv[j];
        }
      }
    }
    __syncthreads();
    const int digit = s_red_i[0];
    krem -= s_red_i[1];
    prefix |= (unsigned long long)digit << shift;
    pmask |= 0xFFull << shift;
    __syncthreads();
  }
  if (tid == 0) { s_T = prefix; s_need = krem; s_vi = -1; }
  __syncthreads();
}

// A victim's physical slot for the free pass: FP16-form entries own theirs (>= 0); a codes
// entry (storage index < nq) holds code slot cs = 2 * slot + half, one half of a packed slot:
// its half is released here (socc) and the slot freed once both halves are (encoded -slot-1).
__device__ __forceinline__ int victim_slot(const Dev& d, size_t base, int slot, bool codes) {
  if (!codes) return slot;
  atomicSub(&d.socc[base + (slot >> 1)], 1);
  return -(slot >> 1) - 1;
}

template <int kT>
__global__ void __launch_bounds__(kT, 1024 / kT)
k3_manage(Dev d, Cfg cf, int32_t* __restrict__ kept_map, int32_t* __restrict__ kept_len,
          const __half* __restrict__ knew, const __half* __restrict__ vnew) {
  const int c = blockIdx.x;
  const int l = c / d.B, b = c % d.B;
  const size_t base = (size_t)c * d.cap;
  const size_t sb = (size_t)c * d.nsid;   // this cache's segment-id space (scnt / sstk)
  const int tid = threadIdx.x;
  K3_STAMP(0);

  __shared__ int s_w[33];
  __shared__ int s_n, s_n8, s_nq, s_ftop, s_stop, s_stopb, s_nseg, s_t, s_status, s_N, s_P;
  __shared__ double s_red_d[64];
  __shared__ int s_red_i[64];
  __shared__ double s_elo, s_ehi;
  __shared__ int s_slo, s_shi;
  __shared__ int s_hist[256];
  __shared__ unsigned long long s_T;
  __shared__ int s_need, s_vi;
  __shared__ int s_vt[6];   // fast path: what the single victim frees (slot, segment)

  if (tid == 0) {
    s_n = d.len[c];
    s_n8 = d.n8[c];
    s_nq = d.nq[c];
    s_ftop = d.ftop[c];
    s_stop = d.stop[c];
    s_stopb = d.stopb[c];
    s_nseg = d.nseg[c];
    s_t = *d.tnext;
    const int att = d.att_len[c];
    s_status = (att == s_n ? 0 : att == -2 ? (kStShape | kStNoAttend) : kStNoAttend) | d.pf_status[c];
    const int tier_high = d.conf[b].tier_high;
    switch (cf.policy) {
      case CKV_POLICY_CONFKV:   // layer_budget + min(P, N) (policy.py:262-263)
        s_N = d.budget[l * 2 + (tier_high ? 0 : 1)];
        s_P = min(cf.P, s_N);
        break;
      case CKV_POLICY_FULL:     // FullCachePolicy._manage (baselines.py:71-77): nothing
        s_N = 0x3fffffff;
        s_P = 0;
        break;
      case CKV_POLICY_SLIDING:  // sliding_window_step: keep the window newest (baselines.py:21-31)
        s_N = cf.param;
        s_P = 0;
        break;
      case CKV_POLICY_HEAVY_HITTER:   // heavy_hitter_step (baselines.py:34-54)
        s_N = cf.param;
        s_P = cf.P;
        break;
      default: {                // matched rate: the recorded count (baselines.py:180-186)
        const int cnt = d.evcnt[c];
        d.evcnt[c] = 0;         // consumed: a step without ckv_set_victims evicts nothing
        s_P = cf.P;
        if (cnt > s_n - s_P) {
          s_status |= kStSchedule;
          s_N = s_n;
        } else {
          s_N = s_n - cnt;
        }
      }
    }
  }
  __syncthreads();
  const int n = s_n;
  if (s_status & kStNoAttend) {
    if (kept_map)
      for (int i = tid; i < n; i += kT) kept_map[base + i] = i;
    if (tid == 0) {
      ckv_layer_record r{n, n, 0, s_n8, n, s_nseg, s_status, s_nq};
      d.rec[c] = r;
      d.qcnt[c] = 0;
      d.ccnt[c] = 0;
      d.newslot[c] = -1;
      if (kept_len) kept_len[c] = n;
    }
    return;
  }

  K3_STAMP(1);
  const bool hh = cf.policy == CKV_POLICY_HEAVY_HITTER;
  const int excess = n - s_N;
  const int cut = n - s_P;
  const bool composite_keys = cf.policy == CKV_POLICY_CONFKV || cf.policy == CKV_POLICY_MATCHED_RECENCY ||
                              cf.policy == CKV_POLICY_MATCHED_ATTENTION;
  const bool fast = composite_keys && excess <= 1 && n <= d.kstage;
  extern __shared__ __align__(16) uint8_t k3s[];
  double* st_ema = reinterpret_cast<double*>(k3s);
  int32_t* st_stp = reinterpret_cast<int32_t*>(st_ema + d.kstage);
  int32_t* st_slot = st_stp + d.kstage;
  int32_t* st_pos = st_slot + d.kstage;
  int32_t* st_seg = st_pos + d.kstage;
  uint8_t* st_seen = reinterpret_cast<uint8_t*>(st_seg + d.kstage);
  int vi_fast = -1;
  if (fast) {
    // ---- one pass: EMA commit (cache.py:172-177) into smem + every array the shift moves,
    // min / max of the candidates (policy.py:80-89) on the committed values ----
    double lo = INFINITY, hi = -INFINITY;
    int slo = 0x7fffffff, shi = -0x7fffffff - 1;
    // the arrays only the shift needs go global -> shared with cp.async (no registers, in flight
    // beside the EMA loads below; visible after the wait + the reductions' barriers)
    for (int i = tid; i < n; i += kT) {
      const uint32_t o = (uint32_t)i * 4u;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(st_slot) + o), "l"(d.slot + base + i) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(st_pos) + o), "l"(d.pos + base + i) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(st_seg) + o), "l"(d.seg + base + i) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    constexpr int kF = kU;       // EMA inputs per thread in flight at once (8 spill at 64 registers)
    for (int i0 = tid; i0 < n; i0 += kF * kT) {
      double a[kF], e[kF];
      uint8_t sn[kF];
      int sp[kF];
#pragma unroll
      for (int u = 0; u < kF; ++u) {
        const int i = i0 + u * kT;
        if (i < n) { a[u] = d.abar[base + i]; e[u] = d.ema[base + i]; sn[u] = d.seen[base + i]; sp[u] = d.stp[base + i]; }
      }
#pragma unroll
      for (int u = 0; u < kF; ++u) {
        const int i = i0 + u * kT;
        if (i < n) {
          const double en = sn[u] ? __dadd_rn(__dmul_rn(cf.lam, e[u]), __dmul_rn(cf.one_m_lam, a[u])) : a[u];
          st_ema[i] = en; st_stp[i] = sp[u]; st_seen[i] = 1;
          if (i < cut) {
            lo = fmin(lo, en); hi = fmax(hi, en);
            slo = min(slo, sp[u]); shi = max(shi, sp[u]);
          }
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    K3_STAMP(2);   // staged loads landed (this thread's)
    if (tid == 0) d.att_len[c] = -1;   // consumed
    if (excess == 1) {
      const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        slo = min(slo, __shfl_xor_sync(0xffffffffu, slo, o));
        shi = max(shi, __shfl_xor_sync(0xffffffffu, shi, o));
      }
      if (lane == 0) { s_red_d[warp] = lo; s_red_d[32 + warp] = hi; s_red_i[warp] = slo; s_red_i[32 + warp] = shi; }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kT / 32; ++w) {
          lo = fmin(lo, s_red_d[w]); hi = fmax(hi, s_red_d[32 + w]);
          slo = min(slo, s_red_i[w]); shi = max(shi, s_red_i[32 + w]);
        }
        lo = fmin(lo, s_red_d[0]); hi = fmax(hi, s_red_d[32]);
        slo = min(slo, s_red_i[0]); shi = max(shi, s_red_i[32]);
        s_elo = lo; s_ehi = hi; s_slo = slo; s_shi = shi;
      }
      __syncthreads();
      K3_STAMP(7);   // min / max reduced
      // ---- composite keys (policy.py:90-100) and the arg-min, lowest index on ties ----
      const double elo = s_elo, ehi = s_ehi;
      const double rlo = (double)s_slo, rhi = (double)s_shi;
      const double eden = __dsub_rn(ehi, elo), rden = __dsub_rn(rhi, rlo);
      unsigned long long best = ~0ull;
      int besti = 0x7fffffff;
      for (int i = tid; i < cut; i += kT) {
        const double ah = (ehi == elo) ? 0.0 : __ddiv_rn(__dsub_rn(st_ema[i], elo), eden);
        const double rh = (rhi == rlo) ? 0.0 : __ddiv_rn(__dsub_rn((double)st_stp[i], rlo), rden);
        const double comp = __dadd_rn(__dmul_rn(cf.alpha, ah), __dmul_rn(cf.one_m_alpha, rh));
        const unsigned long long key = (unsigned long long)__double_as_longlong(comp);
        if (key < best || (key == best && i < besti)) { best = key; besti = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
        if (ob < best || (ob == best && oi < besti)) { best = ob; besti = oi; }
      }
      __shared__ unsigned long long s_bkf[32];
      __shared__ int s_bif[32];
      if (lane == 0) { s_bkf[warp] = best; s_bif[warp] = besti; }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kT / 32; ++w)
          if (s_bkf[w] < best || (s_bkf[w] == best && s_bif[w] < besti)) { best = s_bkf[w]; besti = s_bif[w]; }
        s_vi = besti;
        s_T = best;
        s_need = 0;
      }
      __syncthreads();
      vi_fast = s_vi;
    } else {
      __syncthreads();
    }
  }
  if (!fast) {
  // ---- EMA commit (cache.py:172-177) --------------------------------------------------
  // Heavy hitter: the `ema` column holds the aux channel CUM_ATTENTION instead,
  // cum += head mean (accumulate_attention, baselines.py:57-65). Full / sliding: no attention.
  if (cf.policy == CKV_POLICY_CONFKV || cf.policy >= CKV_POLICY_MATCHED_RANDOM) {
    // kU entries per thread per pass: all loads first, then the stores (the loop is latency-bound)
    for (int i0 = tid; i0 < n; i0 += kU * kT) {
      double a[kU], e[kU];
      uint8_t sn[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kT;
        if (i < n) { a[u] = d.abar[base + i]; e[u] = d.ema[base + i]; sn[u] = d.seen[base + i]; }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kT;
        if (i < n) {
          d.ema[base + i] = sn[u] ? __dadd_rn(__dmul_rn(cf.lam, e[u]), __dmul_rn(cf.one_m_lam, a[u])) : a[u];
          d.seen[base + i] = 1;
        }
      }
    }
  } else if (hh) {
    for (int i = tid; i < n; i += kT) d.ema[base + i] = __dadd_rn(d.ema[base + i], d.abar[base + i]);
  }
  __syncthreads();
  if (tid == 0) d.att_len[c] = -1;   // consumed

  K3_STAMP(2);
  // ---- rank + select (policy.py:80-127) -------------------------------------------------
  // Keys by policy: the composite (Conf-KV, matched recency / attention with alpha 0 / 1);
  // the cumulative attention (heavy hitter, >= 0 so its bits order as u64 too); the storage
  // index (sliding window: the oldest go); 1 everywhere but 0 at the host-drawn victims
  // (matched random). Victims are the `excess` smallest (key, index) pairs in every case.
  if (excess > 0 && !composite_keys) {
    const bool rnd = cf.policy == CKV_POLICY_MATCHED_RANDOM;
    unsigned long long best = ~0ull;
    int besti = 0x7fffffff;
    for (int i = tid; i < cut; i += kT) {
      const unsigned long long key = hh ? (unsigned long long)__double_as_longlong(d.ema[base + i])
                                   : rnd ? 1ull : (unsigned long long)i;
      d.keys[base + i] = key;
      if (key < best || (key == best && i < besti)) { best = key; besti = i; }
    }
    __syncthreads();
    if (rnd)
      for (int v = tid; v < excess; v += kT) d.keys[base + d.vlist[(size_t)c * d.cap + v]] = 0ull;
    const int warp = tid >> 5, lane = tid & 31;
    if (excess == 1 && !rnd) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
        if (ob < best || (ob == best && oi < besti)) { best = ob; besti = oi; }
      }
      __shared__ unsigned long long s_bk2[32];
      __shared__ int s_bi2[32];
      if (lane == 0) { s_bk2[warp] = best; s_bi2[warp] = besti; }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kT / 32; ++w)
          if (s_bk2[w] < best || (s_bk2[w] == best && s_bi2[w] < besti)) { best = s_bk2[w]; besti = s_bi2[w]; }
        s_vi = besti;
        s_T = best;
        s_need = 0;
      }
      __syncthreads();
    } else {
      __syncthreads();   // keys visible
      radix_select<kT>(d, base, cut, excess, s_hist, s_red_i, s_T, s_need, s_vi);
    }
  }
  if (excess > 0 && composite_keys) {
    double lo = INFINITY, hi = -INFINITY;
    int slo = 0x7fffffff, shi = -0x7fffffff - 1;
#pragma unroll 4
    for (int i = tid; i < cut; i += kT) {
      const double e = d.ema[base + i];
      const int s = d.stp[base + i];
      lo = fmin(lo, e); hi = fmax(hi, e);
      slo = min(slo, s); shi = max(shi, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      slo = min(slo, __shfl_xor_sync(0xffffffffu, slo, o));
      shi = max(shi, __shfl_xor_sync(0xffffffffu, shi, o));
    }
    const int warp = tid >> 5, lane = tid & 31;
    if (lane == 0) { s_red_d[warp] = lo; s_red_d[32 + warp] = hi; s_red_i[warp] = slo; s_red_i[32 + warp] = shi; }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < kT / 32; ++w) {
        lo = fmin(lo, s_red_d[w]); hi = fmax(hi, s_red_d[32 + w]);
        slo = min(slo, s_red_i[w]); shi = max(shi, s_red_i[32 + w]);
      }
      lo = fmin(lo, s_red_d[0]); hi = fmax(hi, s_red_d[32]);
      slo = min(slo, s_red_i[0]); shi = max(shi, s_red_i[32]);
      s_elo = lo; s_ehi = hi; s_slo = slo; s_shi = shi;
    }
    __syncthreads();
    const double elo = s_elo, ehi = s_ehi;
    const double rlo = (double)s_slo, rhi = (double)s_shi;
    const double eden = __dsub_rn(ehi, elo), rden = __dsub_rn(rhi, rlo);
    // composite keys; track the arg-min for the single-victim fast path
    unsigned long long best = ~0ull;
    int besti = 0x7fffffff;
    for (int i0 = tid; i0 < cut; i0 += kU * kT) {
      double ev[kU];
      int sv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kT;
        if (i < cut) { ev[u] = d.ema[base + i]; sv[u] = d.stp[base + i]; }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int i = i0 + u * kT;
        if (i < cut) {
          const double ah = (ehi == elo) ? 0.0 : __ddiv_rn(__dsub_rn(ev[u], elo), eden);
          const double rh = (rhi == rlo) ? 0.0 : __ddiv_rn(__dsub_rn((double)sv[u], rlo), rden);
          const double comp = __dadd_rn(__dmul_rn(cf.alpha, ah), __dmul_rn(cf.one_m_alpha, rh));
          const unsigned long long key = (unsigned long long)__double_as_longlong(comp);
          if (excess > 1) d.keys[base + i] = key;   // the radix select's input
          if (key < best || (key == best && i < besti)) { best = key; besti = i; }
        }
      }
    }
    if (excess == 1) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, besti, o);
        if (ob < best || (ob == best && oi < besti)) { best = ob; besti = oi; }
      }
      __shared__ unsigned long long s_bk[32];
      __shared__ int s_bi[32];
      if (lane == 0) { s_bk[warp] = best; s_bi[warp] = besti; }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < kT / 32; ++w)
          if (s_bk[w] < best || (s_bk[w] == best && s_bi[w] < besti)) { best = s_bk[w]; besti = s_bi[w]; }
        s_vi = besti;
        s_T = best;
        s_need = 0;
      }
      __syncthreads();
    } else {
      __syncthreads();   // keys visible
      radix_select<kT>(d, base, cut, excess, s_hist, s_red_i, s_T, s_need, s_vi);
    }
  }

  }   // !fast

  K3_STAMP(3);
  // ---- compaction (cache.py:181-220) over metadata only ---------------------------------
  const int n8_old = s_n8, nq_old = s_nq;
  int n_int8_gone = 0, n_nq_gone = 0;
  if (fast && excess <= 0) {
    // no eviction: the committed EMA back in place
    for (int i = tid; i < n; i += kT) { d.ema[base + i] = st_ema[i]; d.seen[base + i] = 1; }
    if (kept_map)
      for (int i = tid; i < n; i += kT) kept_map[base + i] = i;
  }
  if (excess > 0) {
    const unsigned long long T = s_T;
    const int need = s_need, vi = fast ? vi_fast : s_vi;
    int base_keep = 0, base_vict = 0, base_eq = 0;
    if (fast) {
      // one victim: entries before it keep their place (committed EMA, seen); the ones after it
      // are stored one to the left straight from the staged copy
      for (int i = tid; i < n; i += kT) {
        if (i < vi) {
          d.ema[base + i] = st_ema[i];
          d.seen[base + i] = 1;
        } else if (i > vi) {
          const int j = i - 1;
          d.slot[base + j] = st_slot[i]; d.pos[base + j] = st_pos[i]; d.stp[base + j] = st_stp[i];
          d.ema[base + j] = st_ema[i]; d.seen[base + j] = 1; d.seg[base + j] = st_seg[i];
        } else {
          // the single victim's thread also frees what it held (the general path's victim-order
          // free pass, for one victim): its physical slot -- a codes entry's packed slot once
          // both halves are gone -- and its segment once emptied, claimed as that pass claims
          // them (count 0 -> -1)
          const int sg = st_seg[i], sl = st_slot[i];
          const bool codes = i < nq_old, q8 = i < n8_old;
          int ps = sl, fs = 1, fa = 0, fb = 0;
          if (codes) {
            ps = sl >> 1;
            fs = atomicSub(&d.socc[base + ps], 1) == 1;
            if (fs) d.socc[base + ps] = -1;
          }
          if (d.victims) d.victims[base] = i;
          if (q8 && atomicSub(&d.scnt[sb + sg], 1) == 1) {
            d.scnt[sb + sg] = -1;
            fa = sg < d.smax;
            fb = !fa;
          }
          s_vt[0] = ps; s_vt[1] = fs; s_vt[2] = sg; s_vt[3] = fa; s_vt[4] = fb;
          s_vt[5] = (q8 ? 1 : 0) | (codes ? 2 : 0);
        }
      }
      if (kept_map)
        for (int j = tid; j < n - 1; j += kT) kept_map[base + j] = j < vi ? j : j + 1;
    } else if (vi >= 0) {
      // steady state (one victim): entries before it stay, entries after it shift left by
      // one; chunked so every read of a chunk precedes its writes (dst = src - 1)
      constexpr int kS = 2;   // entries per thread per chunk (fewer barrier round trips)
      for (int ch = vi; ch < n; ch += kS * kT) {
        int slot[kS], pos[kS], stp[kS], sg[kS];
        double ema[kS];
        uint8_t seen[kS];
#pragma unroll
        for (int u = 0; u < kS; ++u) {
          const int i = ch + u * kT + tid;
          slot[u] = 0; pos[u] = 0; stp[u] = 0; sg[u] = -1; ema[u] = 0.0; seen[u] = 0;
          if (i > vi && i < n) {
            slot[u] = d.slot[base + i]; pos[u] = d.pos[base + i]; stp[u] = d.stp[base + i];
            ema[u] = d.ema[base + i]; seen[u] = d.seen[base + i]; sg[u] = d.seg[base + i];
          } else if (i == vi) {
            slot[u] = d.slot[base + i]; sg[u] = d.seg[base + i];
          }
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kS; ++u) {
          const int i = ch + u * kT + tid;
          if (i > vi && i < n) {
            const int j = i - 1;
            d.slot[base + j] = slot[u]; d.pos[base + j] = pos[u]; d.stp[base + j] = stp[u];
            d.ema[base + j] = ema[u]; d.seen[base + j] = seen[u]; d.seg[base + j] = sg[u];
          } else if (i == vi) {
            d.vslot[base] = victim_slot(d, base, slot[u], i < nq_old);
            if (d.victims) d.victims[base] = i;
            const bool q8 = i < n8_old;
            d.vseg[base] = q8 ? sg[u] : -1;
            if (q8) atomicSub(&d.scnt[sb + sg[u]], 1);
            s_red_i[2] = q8 ? 1 : 0;
            s_red_i[3] = i < nq_old ? 1 : 0;
          }
        }
        __syncthreads();
      }
      if (kept_map)
        for (int j = tid; j < n - 1; j += kT) kept_map[base + j] = j < vi ? j : j + 1;
      n_int8_gone = (tid == 0) ? s_red_i[2] : 0;
      n_nq_gone = (tid == 0) ? s_red_i[3] : 0;
    }
    for (int ch = 0; ch < n && vi < 0 && !fast; ch += kT) {
      const int i = ch + tid;
      const bool valid = i < n;
      bool vict = false, eq = false;
      if (valid && i < cut) {
        if (vi >= 0) {
          vict = (i == vi);
        } else {
          const unsigned long long key = d.keys[base + i];
          vict = key < T;
          eq = key == T;
        }
      }
      int eqtot;
      const int eqr = block_scan(eq ? 1 : 0, s_w, eqtot);
      if (eq) vict = (base_eq + eqr) < need;
      const bool keep = valid && !vict;
      int ktot;
      const int kr = block_scan(keep ? 1 : 0, s_w, ktot);
      const int nvalid = min(kT, n - ch);
      int slot = 0, pos = 0, stp = 0, sg = -1;
      double ema = 0.0;
      uint8_t seen = 0;
      if (valid) {
        slot = d.slot[base + i];
        sg = d.seg[base + i];
        if (keep) {
          pos = d.pos[base + i];
          stp = d.stp[base + i];
          ema = d.ema[base + i];
          seen = d.seen[base + i];
        }
      }
      __syncthreads();   // every read of this chunk happens before any write
      if (keep) {
        const int j = base_keep + kr;
        d.slot[base + j] = slot;
        d.pos[base + j] = pos;
        d.stp[base + j] = stp;
        d.ema[base + j] = ema;
        d.seen[base + j] = seen;
        d.seg[base + j] = sg;
        if (kept_map) kept_map[base + j] = i;
      } else if (vict) {
        const int vr = base_vict + (tid - kr);
        d.vslot[base + vr] = victim_slot(d, base, slot, i < nq_old);
        if (d.victims) d.victims[base + vr] = i;   // ascending: the compact kept-index map
        const bool q8 = i < n8_old;
        d.vseg[base + vr] = q8 ? sg : -1;
        if (q8) atomicSub(&d.scnt[sb + sg], 1);
      }
      if (vict && i < n8_old) n_int8_gone++;
      if (vict && i < nq_old) n_nq_gone++;
      __syncthreads();
      base_keep += ktot;
      base_vict += nvalid - ktot;
      base_eq += eqtot;
    }
    if (fast) {
      __syncthreads();   // the victim's s_vt
      if (tid == 0) {
        const int ps = s_vt[0], fs = s_vt[1], sg = s_vt[2], fa = s_vt[3], fb = s_vt[4], g = s_vt[5];
        if (fa) d.sstk[sb + s_stop] = sg;
        if (fb) d.sstk[sb + d.smax + s_stopb] = sg;
        if (fs) d.fstk[base + s_ftop] = ps;
        s_ftop += fs;
        s_stop += fa;
        s_stopb += fb;
        s_nseg -= fa + fb;
        s_n8 = n8_old - (g & 1);
        s_nq = nq_old - ((g >> 1) & 1);
      }
      __syncthreads();
    } else {
    n_int8_gone = block_sum(n_int8_gone, s_w);
    n_nq_gone = block_sum(n_nq_gone, s_w);
    // free emptied segments and physical slots, in victim order (deterministic stack order):
    // segments back to their pool; a victim's slot back to the free stack -- for a codes entry
    // (half of a packed slot) only once both halves are gone (the claim below succeeds once)
    __syncthreads();
    int freed_a = 0, freed_b = 0, freed_s = 0;
    for (int v0 = 0; v0 < excess; v0 += kT) {
      const int v = v0 + tid;
      int fa = 0, fb = 0, fs = 0, sg = -1, ps = 0;
      if (v < excess) {
        sg = d.vseg[base + v];
        if (sg >= 0 && atomicCAS(&d.scnt[sb + sg], 0, -1) == 0) {
          fa = sg < d.smax;
          fb = !fa;
        }
        const int vs = d.vslot[base + v];
        ps = vs >= 0 ? vs : -vs - 1;
        fs = vs >= 0 || atomicCAS(&d.socc[base + ps], 0, -1) == 0;
      }
      int ta, tb, ts;
      const int ra = block_scan(fa, s_w, ta);
      const int rb = block_scan(fb, s_w, tb);
      const int rs = block_scan(fs, s_w, ts);
      if (fa) d.sstk[sb + s_stop + freed_a + ra] = sg;
      if (fb) d.sstk[sb + d.smax + s_stopb + freed_b + rb] = sg;
      if (fs) d.fstk[base + s_ftop + freed_s + rs] = ps;
      freed_a += ta;
      freed_b += tb;
      freed_s += ts;
    }
    if (tid == 0) {
      s_ftop += freed_s;
      s_stop += freed_a;
      s_stopb += freed_b;
      s_nseg -= freed_a + freed_b;
      s_n8 = n8_old - n_int8_gone;
      s_nq = nq_old - n_nq_gone;
    }
    __syncthreads();
    }   // !fast
  } else if (kept_map) {
    for (int i = tid; i < n; i += kT) kept_map[base + i] = i;
  }
  const int len_post = n - max(excess, 0);

  K3_STAMP(4);
  // ---- INT8 window: aged HIGH entries [n8, n8 + m) (quantizer.py:54) --------------------
  // One new segment of the m aged survivors (quantizer.py:61-64). m == 1 (the decode steady
  // state): an id from the single-entry pool -- no scale row, no codes written: its codes
  // (+-127 / 0) and scale (|x|/127) are functions of the entry's resident fp16 row, which K2
  // reads. m > 1: a lossy segment (scale row + in-place codes, K4); from then on every INT8
  // entry is read as codes, so single-entry segments still in fp16 form ([nq, n8)) move to
  // lossy-pool ids and get their scale rows and in-place codes too (K4; a step-number jump
  // after single-entry demotions is the only way there).
  int qcnt = 0;
  __shared__ int s_k4q, s_ns;   // the qcnt K4 sees (K4 appends when > 1); the new row's slot
  if (tid == 0) { d.qcnt[c] = 0; d.ccnt[c] = 0; s_k4q = 0; s_ns = -1; }
  if (cf.quantize) {
    const int n8 = s_n8;
    const int lim = s_t - cf.W;
    int cnt = 0;
    for (int j = n8 + tid; j < len_post; j += kT) cnt += (d.stp[base + j] <= lim) ? 1 : 0;
    qcnt = block_sum(cnt, s_w);
    if (qcnt > 0) {
      __shared__ int s_sslot, s_cv;
      if (tid == 0) {
        s_sslot = -1;
        s_cv = 0;
        if (qcnt == 1) {
          s_sslot = d.sstk[sb + d.smax + (--s_stopb)];   // never empty: nsid - smax = cap ids
        } else {
          const int cv = n8 - s_nq;
          if (s_stop < cv + 1) {
            s_status |= kStSegOverflow;
          } else {
            s_cv = cv;
            s_sslot = d.sstk[sb + (s_stop - 1 - cv)];
          }
        }
      }
      __syncthreads();
      const int ss = s_sslot, cv = s_cv, nq0 = s_nq;
      for (int k = tid; k < cv; k += kT) {   // single-entry segments -> lossy-pool ids
        const int j = nq0 + k;
        const int old = d.seg[base + j];
        const int nw = d.sstk[sb + (s_stop - 1 - k)];
        d.seg[base + j] = nw;
        d.scnt[sb + nw] = 1;
        d.scnt[sb + old] = 0;
        d.sstk[sb + d.smax + s_stopb + k] = old;
      }
      if (ss >= 0)
        for (int j = n8 + tid; j < n8 + qcnt; j += kT) d.seg[base + j] = ss;
      if (ss >= 0 && qcnt > 1) {
        // codes take half a slot: aged entries pair up (n8 + 2k, n8 + 2k + 1) in the slot of
        // the first, whose 2*D-byte head rows hold both code rows (code slots 2s, 2s + 1); the
        // second's slot is freed after K4 has read its fp16 rows (old slot kept in vseg)
        for (int k = tid; 2 * k < qcnt; k += kT) {
          const int ja = n8 + 2 * k, sa = d.slot[base + ja];
          d.slot[base + ja] = 2 * sa;
          const bool pair = 2 * k + 1 < qcnt;
          d.socc[base + sa] = pair ? 2 : 1;
          if (pair) {
            const int sbv = d.slot[base + ja + 1];
            d.slot[base + ja + 1] = 2 * sa + 1;
            d.vseg[base + k] = sbv;
            d.fstk[base + s_ftop + k] = sbv;
          }
        }
        for (int k = tid; k < cv; k += kT) {   // converted single-entry segments: unpacked half
          const int sa = d.slot[base + nq0 + k];
          d.slot[base + nq0 + k] = 2 * sa;
          d.socc[base + sa] = 1;
        }
      }
      __syncthreads();
      if (tid == 0 && ss >= 0) {
        d.scnt[sb + ss] = qcnt;
        s_nseg += 1;
        if (qcnt > 1) {
          s_stop -= cv + 1;
          s_stopb += cv;
          s_nq = n8 + qcnt;
          s_ftop += qcnt / 2;
          d.clo[c] = nq0;
          d.ccnt[c] = cv;
        }
        d.qlo[c] = n8;
        d.qcnt[c] = qcnt;
        s_k4q = qcnt;
        d.qseg[c] = ss;
        s_n8 = n8 + qcnt;
      }
    }
  }
  __syncthreads();

  K3_STAMP(5);
  // ---- append metadata (cache.py:111-132; policy.py:203-206) ----------------------------
  if (tid == 0) {
    int len_after = len_post;
    if (s_ftop == 0) {
      s_status |= kStOverflow;
      d.newslot[c] = -1;
    } else {
      const int ps = d.fstk[base + (--s_ftop)];
      const int j = len_post;
      d.slot[base + j] = ps;
      d.pos[base + j] = cf.prefill_len + s_t - 1;
      d.stp[base + j] = s_t;
      d.ema[base + j] = 0.0;
      d.seen[base + j] = 0;
      d.seg[base + j] = -1;
      d.newslot[c] = ps;
      len_after = len_post + 1;
    }
    d.len[c] = len_after;
    d.n8[c] = s_n8;
    d.nq[c] = s_nq;
    d.ftop[c] = s_ftop;
    d.stop[c] = s_stop;
    d.stopb[c] = s_stopb;
    d.nseg[c] = s_nseg;
    ckv_layer_record r{n, len_post, max(excess, 0), s_n8, len_after, s_nseg, s_status, s_nq};
    d.rec[c] = r;
    if (kept_len) kept_len[c] = len_post;
    if (len_after > len_post) s_ns = d.newslot[c];
  }
  // ---- append K/V rows (cache.py:111-132): here unless a lossy demotion is pending (its codes
  // rewrite in K4 frees slots the new row may take, so K4 appends after it). The new token's
  // rows of all KV heads are one contiguous Hkv*D run on both sides: 16-byte vectors.
  __syncthreads();
  if (knew && s_k4q <= 1) {
    const int ns = s_ns;
    if (ns >= 0) {
      const size_t row = (size_t)d.Hkv * d.D;
      if (((reinterpret_cast<uintptr_t>(knew) | reinterpret_cast<uintptr_t>(vnew)) & 15) == 0) {
        const int nv = (int)(row / 8);   // 8 halfs per vector (D is a multiple of 16)
        for (int k = tid; k < 2 * nv; k += kT) {
          const int isv = k >= nv, e = isv ? k - nv : k;
          const uint4* src = reinterpret_cast<const uint4*>((isv ? vnew : knew) + (size_t)c * row) + e;
          uint4* dst = reinterpret_cast<uint4*>((isv ? d.vf : d.kf) + (base + ns) * row) + e;
          *dst = __ldg(src);
        }
      } else {
        for (int k = tid; k < 2 * (int)row; k += kT) {
          const int isv = k >= (int)row, e = isv ? k - (int)row : k;
          (isv ? d.vf : d.kf)[(base + ns) * row + e] = (isv ? vnew : knew)[(size_t)c * row + e];
        }
      }
    }
  }
  K3_STAMP(6);
}

// K4: INT8 demotion (quantize_segment, quantizer.py:16-34) and the K/V half of append. One
// CTA per (KV head, cache).
//   Lossy segment [qlo, qlo + qcnt): per-(K|V, dim) lane amax over the aged rows, scale =
//   amax/127 in IEEE fp32 into the segment's scale row; then the codes are written IN PLACE
//   over the first D bytes of each aged row's 2*D-byte fp16 head row (the fp16 values are not
//   needed once the entry is lossy): one warp per (row, K|V), every lane loads its dims,
//   __syncwarp, then stores their codes (a code byte overlays the fp16 of a lower dim).
//   Single-entry segments turned lossy-form [clo, clo + ccnt): the same, with each row's own
//   scale |x|/127 written to its segment's scale row.
//   A single-entry demotion (the decode steady state) writes nothing: its codes (+-127 / 0)
//   and scale (|x|/127) are functions of the resident fp16 row.
constexpr int kQThreads = 256;

__device__ __forceinline__ float quant_code(float x, float scale) {   // quantizer.py:28-33
  const float safe = scale > 0.f ? scale : 1.0f;
  const float s = __fdiv_rn(x, safe);
  float code = copysignf(floorf(__fadd_rn(fabsf(s), 0.5f)), s);
  code = fminf(fmaxf(code, -127.f), 127.f);
  return scale > 0.f ? code : 0.f;                    // all-zero lanes -> 0 (quantizer.py:33)
}

// Physical fp16 slot of aged entry j of a lossy segment starting at qlo (before K3 packed it):
// the first of a pair keeps its slot (code slot 2s), the second's old slot is in vseg.
__device__ __forceinline__ int aged_slot(const Dev& d, size_t base, int qlo, int j) {
  const int k = j - qlo;
  return (k & 1) ? d.vseg[base + (k >> 1)] : (d.slot[base + j] >> 1);
}

// Codes of one (entry, K|V) row: the lane's dims of the fp16 row at `src`, written as bytes
// at `dst` (both in the same 2*D-byte head row for the first entry of a pair or a converted
// one): every lane reads before any lane writes.
template <bool CONVERT>
__device__ __forceinline__ void codes_rows(const Dev& d, int c, int h, int lo, int cnt, const float* s_scale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int D = d.D;
  const size_t base = (size_t)c * d.cap;
  const size_t row = (size_t)d.Hkv * D;
  // lossy segment: one warp per (pair, K|V) -- both entries' fp16 rows are read before the
  // pair's slot row is overwritten; converted single-entry segments: one warp per (entry, K|V)
  const int units = CONVERT ? cnt : (cnt + 1) / 2;
  for (int p = warp; p < 2 * units; p += nw) {
    const int u = p >> 1, isv = p & 1;
    __half* kv = isv ? d.vf : d.kf;
    const int ja = lo + (CONVERT ? u : 2 * u);
    const bool pair = !CONVERT && 2 * u + 1 < cnt;
    const int sa = CONVERT ? (d.slot[base + ja] >> 1) : aged_slot(d, base, lo, ja);
    __half* ra = kv + (base + sa) * row + (size_t)h * D;
    const __half* rb = pair ? kv + (base + d.vseg[base + u]) * row + (size_t)h * D : nullptr;
    float xa[4], xb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int dd = lane + 32 * k;
      xa[k] = dd < D ? __half2float(ra[dd]) : 0.f;
      xb[k] = (pair && dd < D) ? __half2float(rb[dd]) : 0.f;
    }
    __syncwarp();                                     // the row is read before its bytes are reused
    int8_t* cr = reinterpret_cast<int8_t*>(ra);       // code slots 2*sa (bytes [0, D)), 2*sa + 1 ([D, 2D))
    float* srow = nullptr;
    if (CONVERT) srow = (isv ? d.vsc : d.ksc) + (((size_t)c * d.smax + d.seg[base + ja]) * d.Hkv + h) * D;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int dd = lane + 32 * k;
      if (dd < D) {
        float sc;
        if (CONVERT) {
          sc = __fdiv_rn(fabsf(xa[k]), 127.0f);       // the single member's amax / 127
          srow[dd] = sc;
        } else {
          sc = s_scale[isv * D + dd];
        }
        cr[dd] = (int8_t)(int)quant_code(xa[k], sc);
        if (pair) cr[D + dd] = (int8_t)(int)quant_code(xb[k], sc);
      }
    }
  }
}

__global__ void __launch_bounds__(kQThreads)
k4_quant_append(Dev d, const __half* __restrict__ knew, const __half* __restrict__ vnew) {
  K4_STAMP(0);
  const int h = blockIdx.x, c = blockIdx.y;
  const int D = d.D;
  const int lanes = 2 * D;
  const int tgs = max(1, kQThreads / lanes);
  const int lane = threadIdx.x % lanes, tg = threadIdx.x / lanes;
  const bool active = tg < tgs && threadIdx.x < tgs * lanes;
  const int isv = lane / D, dd = lane % D;
  const size_t row = (size_t)d.Hkv * D;
  const size_t base = (size_t)c * d.cap;
  const int qcnt = d.qcnt[c], ccnt = d.ccnt[c];
  if (qcnt <= 1) {   // no codes to write (ccnt > 0 only beside a lossy demotion); K3 appended
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *d.tnext += 1;
    K4_STAMP(1);
    return;
  }
  __shared__ float s_amax[kQThreads];
  if (qcnt > 1) {
    const int qlo = d.qlo[c], qseg = d.qseg[c];
    const __half* src = isv ? d.vf : d.kf;
    float amax = 0.f;
    if (active) {
      for (int j = qlo + tg; j < qlo + qcnt; j += tgs)
        amax = fmaxf(amax, fabsf(__half2float(src[(base + aged_slot(d, base, qlo, j)) * row + (size_t)h * D + dd])));
    }
    s_amax[threadIdx.x] = amax;
    __syncthreads();
    if (active && tg == 0) {
      for (int k = 1; k < tgs; ++k) amax = fmaxf(amax, s_amax[k * lanes + lane]);
      const float scale = __fdiv_rn(amax, 127.0f);   // amax / 127 in fp32
      (isv ? d.vsc : d.ksc)[(((size_t)c * d.smax + qseg) * d.Hkv + h) * D + dd] = scale;
      s_amax[lane] = scale;                           // lanes [0, 2D): the scale rows
    }
    __syncthreads();
    codes_rows<false>(d, c, h, qlo, qcnt, s_amax);
  }
  if (ccnt > 0) codes_rows<true>(d, c, h, d.clo[c], ccnt, nullptr);
  __syncthreads();   // the pairs' freed slots are read before the append may reuse one
  // append this KV head's row of the new token
  const int ns = d.newslot[c];
  if (ns >= 0 && knew) {
    for (int k = threadIdx.x; k < 2 * D; k += blockDim.x) {
      const int v = k / D, e = k % D;
      const __half* s = v ? vnew : knew;
      __half* t = v ? d.vf : d.kf;
      t[(base + ns) * row + (size_t)h * D + e] = s[((size_t)c * d.Hkv + h) * D + e];
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *d.tnext += 1;
  K4_STAMP(1);
}

// Prefill: metadata + physical slot allocation (one CTA per cache) ...
__global__ void k_prefill_meta(Dev d, int c0, int n, int first_pos, int prefill_len) {
  const int c = c0 + blockIdx.x;
  const size_t base = (size_t)c * d.cap;
  const int len = d.len[c], ftop = d.ftop[c];
  const bool fits = len + n <= d.cap && ftop >= n;
  for (int i = threadIdx.x; i < n && fits; i += blockDim.x) {
    const int j = len + i;
    d.slot[base + j] = d.fstk[base + ftop - 1 - i];
    d.pos[base + j] = first_pos + i;
    d.stp[base + j] = first_pos + i - prefill_len;
    d.ema[base + j] = 0.0;
    d.seen[base + j] = 0;
    d.seg[base + j] = -1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (fits) {
      d.pf_base[c] = len;
      d.len[c] = len + n;
      d.ftop[c] = ftop - n;
    } else {
      d.pf_base[c] = -1;
      d.rec[c].status |= kStOverflow;
      d.pf_status[c] |= kStOverflow;   // sticky: every later step reports it (the entries are lost)
    }
  }
}

// ... then the K/V rows, 16 bytes per thread.
__global__ void k_prefill_data(Dev d, int c0, const __half* __restrict__ k, const __half* __restrict__ v,
                               int n) {
  const int c = c0 + blockIdx.y;
  const int pb = d.pf_base[c];
  if (pb < 0) return;
  const size_t base = (size_t)c * d.cap;
  const int vec_per_tok = d.Hkv * d.D / 8;
  const size_t total = (size_t)n * vec_per_tok;
  const size_t row = (size_t)d.Hkv * d.D;
  const uint4* ks = reinterpret_cast<const uint4*>(k + (size_t)(c - c0) * n * row);
  const uint4* vs = reinterpret_cast<const uint4*>(v + (size_t)(c - c0) * n * row);
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx / vec_per_tok), r = (int)(idx % vec_per_tok);
    const int ps = d.slot[base + pb + i];
    reinterpret_cast<uint4*>(d.kf + (base + ps) * row)[r] = ks[idx];
    reinterpret_cast<uint4*>(d.vf + (base + ps) * row)[r] = vs[idx];
  }
}

__global__ void k_init(Dev d) {
  const int c = blockIdx.x;
  const size_t base = (size_t)c * d.cap;
  for (int k = threadIdx.x; k < d.cap; k += blockDim.x) d.fstk[base + k] = d.cap - 1 - k;
  for (int k = threadIdx.x; k < d.nsid; k += blockDim.x) {
    // pop order: ids 0, 1, ... of each pool
    d.sstk[(size_t)c * d.nsid + k] = k < d.smax ? d.smax - 1 - k : d.smax + d.nsid - 1 - k;
    d.scnt[(size_t)c * d.nsid + k] = 0;
  }
  if (threadIdx.x == 0) {
    d.len[c] = 0; d.n8[c] = 0; d.nq[c] = 0; d.ftop[c] = d.cap; d.stop[c] = d.smax; d.stopb[c] = d.cap;
    d.nseg[c] = 0; d.ccnt[c] = 0;
    d.att_len[c] = -1; d.qcnt[c] = 0; d.newslot[c] = -1; d.pf_base[c] = -1; d.pf_status[c] = 0;
    ckv_layer_record r{0, 0, 0, 0, 0, 0, 0, 0};
    d.rec[c] = r;
    if (c == 0) *d.tnext = 1;
    if (c < d.B) d.ticket[c] = 0;
  }
}

__global__ void k_set_step(Dev d, int t) { *d.tnext = t; }

}  // namespace

cudaError_t launch_manage(const Dev& d, const Cfg& c, const __half* knew, const __half* vnew,
                          int32_t* kept_map, int32_t* kept_len, cudaStream_t s) {
  const size_t sm = (size_t)kStageBytes(d.kstage);
  static size_t configured = 0;
  static int nsm = 0;
  if (sm > configured) {
    cudaError_t ea = cudaFuncSetAttribute(k3_manage<kTBig>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (ea == cudaSuccess)
      ea = cudaFuncSetAttribute(k3_manage<kTBig / 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (ea != cudaSuccess) return ea;
    configured = sm;
  }
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // More caches than two 512-thread CTAs per SM hold (a second wave) but short enough that four
  // staged CTAs fit an SM's shared memory: 256-thread CTAs, one wave (CKV_K3T=512|256 forces)
  const bool small = d.k3t_force ? d.k3t_force == kTBig / 2
                             : d.C > 2 * nsm && 4 * (sm + 4096) <= 220 * 1024;
  if (small) k3_manage<kTBig / 2><<<d.C, kTBig / 2, sm, s>>>(d, c, kept_map, kept_len, knew, vnew);
  else k3_manage<kTBig><<<d.C, kTBig, sm, s>>>(d, c, kept_map, kept_len, knew, vnew);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k4_quant_append<<<dim3(d.Hkv, d.C), kQThreads, 0, s>>>(d, knew, vnew);
  return cudaGetLastError();
}

cudaError_t launch_set_step(const Dev& d, int t, cudaStream_t s) {
  k_set_step<<<1, 1, 0, s>>>(d, t);
  return cudaGetLastError();
}

cudaError_t launch_prefill(const Dev& d, const Cfg& c, int c0, int ccount, const __half* k,
                           const __half* v, int n, int first_pos, cudaStream_t s) {
  k_prefill_meta<<<ccount, 256, 0, s>>>(d, c0, n, first_pos, c.prefill_len);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t total = (size_t)n * d.Hkv * d.D / 8;
  const int bx = (int)std::min<size_t>((total + 255) / 256, 1024);
  k_prefill_data<<<dim3(std::max(bx, 1), ccount), 256, 0, s>>>(d, c0, k, v, n);
  return cudaGetLastError();
}

cudaError_t launch_init(const Dev& d, cudaStream_t s) {
  k_init<<<d.C, 256, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace ckv

#ifdef CKV_TRACE
extern "C" int ckv_debug_k4trace(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(ckv::g_k4trace) ? bytes : sizeof(ckv::g_k4trace);
  return (int)cudaMemcpyFromSymbol(host, ckv::g_k4trace, n);
}
extern "C" int ckv_debug_k3trace(void* host, size_t bytes) {
  const size_t n = bytes < sizeof(ckv::g_k3trace) ? bytes : sizeof(ckv::g_k3trace);
  return (int)cudaMemcpyFromSymbol(host, ckv::g_k3trace, n);
}
#endif
