// Internal device-state layout shared by the kernels and the ABI layer.
//
// HBM layout (C = num_layers * batch caches, cache c = layer * batch + seq):
//   kf, vf   half  [C][cap][Hkv][D]   physical token slots holding fp16 rows: FP16 entries and
//                                     single-entry INT8 segments (whose codes +-127 / 0 and
//                                     scale |x|/127 are functions of the row). Entries of lossy
//                                     (multi-member) segments hold only their int8 codes, two
//                                     entries per slot: code slot cs = 2*slot + half, the code
//                                     row of KV head h at byte ((c*cap + slot)*Hkv + h)*2D +
//                                     half*D -- kq / vq view kf / vf as [C*cap*Hkv*2][D] bytes
//   slot     i32   [C][cap]           logical storage index -> physical slot
//   pos/stp  i32   [C][cap]           original position / generation step
//   ema      f64   [C][cap], seen u8 [C][cap], seg i32 [C][cap] (-1 = HIGH)
//   ksc,vsc  f32   [C][smax][Hkv][D]  scales of the lossy segments (segment ids [0, smax))
//   scnt     i32   [C][smax + cap]    member count per segment id; ids [smax, smax + cap) are
//                                     single-entry segments (no scale row)
// Logical order is the reference's storage order (sorted by position); INT8
// entries are always the logical prefix [0, n8) because aging is monotone in
// generation step (quantizer.py:54) and compaction preserves order; entries read
// as codes are the prefix [0, nq) of that.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/confkv_b200.h"

namespace ckv {

constexpr int kSplitTokens = 512;   // K2 split-K chunk (entries per CTA)
constexpr int kAbsorbTokens = 64;   // a trailing partial split of <= this many FP16 entries joins the split before it
constexpr int kConfThreads = 256;   // K1 block
constexpr int kConfVec = 4;         // K1 elements per vector load (f32)
constexpr int kConfIters = 4;       // K1 vectors per thread per block (loads issued together)
constexpr int kConfPerBlock = kConfThreads * kConfVec * kConfIters;
constexpr int kManageThreads = 512;   // K3 block: 2 CTAs per SM fit the register file (1024 did not: two waves)

struct Dev {
  int L, B, Hq, Hkv, D, V, G, cap, smax, C, nsplit;
  int nsid;                             // segment ids per cache: smax (lossy, with scales) + cap (single-entry)
  // K2 partials: split s has two parts, slot 2s = entries [s*512, cut) read as INT8 codes and
  // slot 2s+1 = [cut, end) read as FP16 rows, cut = clamp(nq, s*512, end) when cut_nq (INT8 on,
  // D = 128: codes parts run on the tcgen05 kernel), else cut = end (whole split in slot 2s).
  int npart, cut_nq;
  int sld;                              // K2 score scratch row stride (cap rounded up to 64)
  int quant;                            // INT8 window on (cfg.quantize)
  int gen_splits;                       // host estimate of non-bulk splits per cache (launch width)
  int dyn_items;                        // K2 persistent grid claims items dynamically (small launches)
  int use_tc;                           // host: this launch runs the persistent tcgen05 grid
  int fstream;                          // FP16 parts run on the streaming kernel (k2_fp16_stream)
  int scodes;                           // ... and single-segment codes parts too (no tcgen05 grid, D = 128)
  int live_splits;                      // host bound on 512-entry splits any cache holds now (<= nsplit)
  int absorb;                           // K2 (mma path): trailing remainder of <= kAbsorbTokens FP16 entries
                                        // is read by the last full split (its own split is empty)
  // K2 path forcing (tests / A-B; read from CKV_COMB / CKV_DYN at ckv_create): comb_force
  // -1 auto, 0 k2_combine<1>, 1 k2_combine<4>, 2 k2_combine_staged; dyn_force -1 auto,
  // 0 static-stride items, 1 dynamic item claims in the persistent tcgen05 grid
  int comb_force, dyn_force;
  int fs_force;                         // CKV_FSTREAM: -1 auto, 0 / 1 FP16 parts off / on the streaming kernel
  int k3t_force;                        // CKV_K3T: 0 auto, 512 / 256 K3 threads per CTA
  int gen_cap;                          // CKV_GENCAP (default 1): one wave of general CTAs when the stream takes codes parts
  int kstage;                           // K3 staged fast path: caches of <= kstage entries (min(cap, kStage))
  __half *kf, *vf;
  int8_t *kq, *vq;                      // == kf / vf viewed as [C*cap*Hkv*2][D] code rows (code_row)
  int32_t *slot, *pos, *stp;
  double* ema;
  uint8_t* seen;
  int32_t* seg;
  int32_t *len, *n8;
  // nq: logical prefix K2 must read as INT8 codes. Entries in [nq, n8) belong to segments
  // quantised from a single entry, whose dequantised value 127*fl(|x|/127) equals the resident
  // FP16 row x but for 214 fp16 magnitudes (1 fp32 ulp), so K2 reads those rows as FP16.
  int32_t* nq;
  int32_t *fstk, *ftop;                 // free physical slots (stack)
  int32_t* socc;                        // [C][cap] codes halves live in a packed slot (codes entries)
  int32_t* vslot;                       // [C][cap] K3 scratch: this step's victims' slots
  int32_t* victims;                     // optional [C][cap] output: this step's evicted storage indices,
                                        // ascending (ckv_victims_out; the kept map's complement)
  float *ksc, *vsc;
  int32_t *scnt, *sstk, *stop, *nseg;   // segment pool: member count, free stacks (ids [0, smax) at
                                        // sstk[c*nsid + ...], top stop; ids [smax, nsid) at
                                        // sstk[c*nsid + smax + ...], top stopb)
  int32_t* stopb;
  float *score, *pm, *pz, *po;          // K2 scratch
  double* abar;                         // staged head-mean attention [C][cap]
  int32_t* att_len;                     // n seen by the staged attention (-1: none, -2: rows of the
                                        // wrong length were staged, cache.py:164-167)
  int32_t* pf_status;                   // sticky prefill status (kStOverflow), ORed into every record
  double* cpart;                        // K1 block partials [B][nblk][8]
  int32_t* ticket;                      // K1 last-block tickets [B]
  int32_t* k1exit;                      // K1 grid exit ticket (the last CTA waits for the prerequisite grid)
  ckv_seq_record* conf;                 // [B]
  uint64_t* keys;                       // K3 composite keys [C][cap]
  int32_t* vseg;                        // K3 victim segment list [C][cap]
  int32_t *qlo, *qcnt, *qseg, *newslot; // K3 -> K4 plan [C]
  int32_t *clo, *ccnt;                  // K3 -> K4: single-entry segments [clo, clo+ccnt) turned lossy-form
  int32_t* pf_base;                     // prefill base index [C]
  ckv_layer_record* rec;                // [C]
  int32_t* budget;                      // [L][2]
  int32_t* tnext;                       // device step counter
  int32_t* work;                        // K2 persistent grid's dynamic item counter (reset by k2_combine)
  int32_t* evcnt;                       // matched-rate: this step's eviction count [C]
  int32_t* vlist;                       // matched-rate random: victim indices [C][cap]
};

// Row of code slot cs (KV head h, cache base c*cap) in the [C*cap*Hkv*2][D]-byte view kq / vq.
__host__ __device__ __forceinline__ int code_row(size_t ccap, int cs, int Hkv, int h) {
  return (int)(((ccap + (size_t)(cs >> 1)) * Hkv + h) * 2 + (cs & 1));
}

// TMA descriptors over the K/V stores viewed as 2-D [C*cap*Hkv rows][D]: one
// row = one KV head of one physical slot; one-row boxes, used with gather4.
// *_sw: 128B-swizzled variants (box <= 128 bytes: 64 fp16 / D int8 columns)
// feeding the tensor-core consumer's bank-conflict-free smem layout.
struct Maps {
  CUtensorMap kf, vf, kq, vq;
  CUtensorMap kf_sw, vf_sw, kq_sw, vq_sw;
};

struct Cfg {
  double tau, alpha, one_m_alpha, lam, one_m_lam, wH, wM, wP, temperature;
  int P, W, quantize, temp_mode, prefill_len;
  int policy, param;                    // CKV_POLICY_*, window / cap
};

enum StatusBits : int32_t {
  kStNonFinite = 1,      // non-finite logits (confidence.py:36-37)
  kStNoAttend = 2,       // manage without a matching attend/stage (policy.py:195-196)
  kStOverflow = 4,       // capacity exhausted (reference would grow, cache.py:120-121)
  kStSegOverflow = 8,    // INT8 segment pool exhausted
  kStStepMismatch = 16,
  kStSchedule = 32,      // matched-rate count above the candidates (baselines.py:165-168)
  kStShape = 64,         // staged attention rows do not match valid_len (cache.py:164-167)
};

// Kernel launchers (defined in the k*.cu files). Return cudaError_t.
cudaError_t launch_confidence(const Dev& d, const Cfg& c, const void* logits, int dtype, int64_t ld,
                              cudaStream_t s, int voff = 0, double* partial_out = nullptr, bool pdl = false);
cudaError_t launch_confidence_merge(const Dev& d, const Cfg& c, const double* parts, int shards, int64_t vtotal,
                                    cudaStream_t s);
cudaError_t launch_stage_weights(const Dev& d, int c0, int ccount, const float* w, int shards, cudaStream_t s);
// K1 arguments for launch_attend to run the confidence pass inline (between the attention grids
// and the combine, programmatic dependent launches) when the tcgen05 grid fills the GPU;
// `inlined` reports whether it did.
struct K1Inline {
  const Cfg* c;
  const void* logits;
  int dtype;
  int64_t ld;
  int inlined;
};
cudaError_t launch_attend(const Dev& d, const Maps& maps, int c0, int ccount, const __half* q,
                          float* out, float* wdump, cudaStream_t s, cudaEvent_t mid = nullptr,
                          K1Inline* k1 = nullptr);
cudaError_t launch_stage_rows(const Dev& d, int layer, const double* rows, int ld, cudaStream_t s);
cudaError_t launch_head_partial(const Dev& d, int c0, int ccount, const float* w, const double* acc_in, double* acc_out,
                                cudaStream_t s);
cudaError_t launch_stage_mass(const Dev& d, int c0, int ccount, const double* acc, int total_heads, cudaStream_t s);
cudaError_t launch_manage(const Dev& d, const Cfg& c, const __half* knew, const __half* vnew,
                          int32_t* kept_map, int32_t* kept_len, cudaStream_t s);
cudaError_t launch_prefill(const Dev& d, const Cfg& c, int c0, int ccount, const __half* k,
                           const __half* v, int n, int first_pos, cudaStream_t s);
cudaError_t launch_init(const Dev& d, cudaStream_t s);
cudaError_t launch_set_step(const Dev& d, int t, cudaStream_t s);
bool attend_supported(int D, int G);
int last_attend_launches();   // kernels the last launch_attend issued on this thread

}  // namespace ckv
