/*
 * confkv_b200.h — C ABI of the B200-native Conf-KV cache-manager hot path.
 *
 * Drop-in boundary for the reference's per-step cache manager
 * (`/root/reference/pkg/src/confkv`, a CPU Python/NumPy package). Each entry
 * point names the reference interface it replaces. All calls:
 *   - take plain device pointers, sizes and a `cudaStream_t` passed as void*;
 *   - are asynchronous on that stream, never synchronise, never throw;
 *   - return an int status (CKV_OK = 0, negative = error, see below) and leave
 *     a message for ckv_last_error();
 *   - must be serialised per engine (single owner, like LayerCache,
 *     cache.py:49-54); distinct engines are independent.
 * Data-dependent failures that can only be seen on the device (non-finite
 * logits, capacity overflow, a step without its attend) are recorded in the
 * per-step records and surfaced by ckv_read_records().
 *
 * Layout conventions (row-major, innermost last):
 *   fp16 K/V/q      IEEE binary16, uint16 storage
 *   q               [layer_count][batch][num_heads][head_dim]
 *   k_new, v_new    [num_layers][batch][num_kv_heads][head_dim]
 *   prefill k/v     [layer_count][batch][n][num_kv_heads][head_dim]
 *   out             [layer_count][batch][num_heads][head_dim] fp32
 *   logits          [batch][ld] fp32, bf16 or fp64, first vocab_size entries used
 *   kept_map        [num_layers][batch][capacity] int32 (old storage index of
 *                   survivor j, j < kept_len[l][b])
 */
#ifndef CONFKV_B200_H
#define CONFKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKV_OK 0
#define CKV_EINVAL -1    /* ValueError   (shape / argument errors)          */
#define CKV_ECONFIG -2   /* ConfigError  (config.py:16)                     */
#define CKV_ERUNTIME -3  /* RuntimeError (state misuse, e.g. missing attend) */
#define CKV_ECUDA -4     /* CUDA launch / allocation failure                */
#define CKV_ENOMEM -5    /* device memory exhausted                         */

#define CKV_DTYPE_F32 0
#define CKV_DTYPE_BF16 1
#define CKV_DTYPE_F64 2   /* the reference's float64 logits (confidence.py:31-39) */

/* Policy knobs, PolicyConfig field for field (config.py:42-58). The pyramid
 * fields are consumed on the host into `budget_table` (policy.py:130-137,
 * 249-254); sampling is greedy or temperature (confidence only). */
typedef struct ckv_config {
  double tau;
  int32_t n_high, n_low, protected_p, fp16_window_w, block_size_b;
  double alpha, ema_lambda;
  double w_entropy, w_margin, w_top;
  int32_t quantize;          /* ConfKVEngine(quantize=...) policy.py:239 */
  int32_t temperature_mode;  /* sampling_mode == "temperature"           */
  double temperature;
  /* Which policy's _manage runs in ckv_manage (baselines.py:68-191 for the
   * comparison policies; those never quantize). policy_param = the sliding
   * window (SlidingWindowPolicy.window) or the heavy-hitter cap. */
  int32_t policy;            /* CKV_POLICY_*                              */
  int32_t policy_param;
} ckv_config;

#define CKV_POLICY_CONFKV 0             /* ConfKVEngine (policy.py:230-274)              */
#define CKV_POLICY_FULL 1               /* FullCachePolicy: no eviction, no EMA          */
#define CKV_POLICY_SLIDING 2            /* SlidingWindowPolicy: keep the newest window   */
#define CKV_POLICY_HEAVY_HITTER 3       /* HeavyHitterPolicy: cumulative attention + P   */
#define CKV_POLICY_MATCHED_RANDOM 4     /* MatchedRatePolicy(mode="random")              */
#define CKV_POLICY_MATCHED_RECENCY 5    /* MatchedRatePolicy(mode="recency_only")        */
#define CKV_POLICY_MATCHED_ATTENTION 6  /* MatchedRatePolicy(mode="attention_only")      */

/* ModelShape (config.py:20-32) plus the GQA KV-head count. */
typedef struct ckv_shape {
  int32_t num_layers, num_heads, num_kv_heads, head_dim, vocab_size;
} ckv_shape;

/* One StepRecord field set for one (layer, sequence) (policy.py:36-69).
 * int8_codes: leading INT8 entries the next attend reads as codes + segment scales; the other
 * int8_count - int8_codes INT8 entries belong to single-entry segments (codes +-127 / 0, scale
 * |x|/127) and are read from their resident FP16 rows x, which equal code*scale except for 214
 * of the 31,743 positive finite fp16 magnitudes (one fp32 ulp apart). */
typedef struct ckv_layer_record {
  int32_t len_pre, len_post, evicted, int8_count, len_after, num_segments, status, int8_codes;
} ckv_layer_record;

/* Confidence features + budget + token for one sequence (confidence.py:22-28). */
typedef struct ckv_seq_record {
  double score, entropy_norm, margin, margin_sig, top_prob;
  int32_t tier_high, token, status, pad;
} ckv_seq_record;

typedef struct ckv_engine ckv_engine;

/* Thread-local text of the last failing call. */
const char* ckv_last_error(void);
/* Library/ABI version (major*10000 + minor*100 + patch). */
int ckv_version(void);

/* ConfKVEngine.__init__ (policy.py:235-247) for `batch` independent sequences.
 * `budget_table` = host int32[num_layers][2]: budget when confident / when
 * uncertain per layer. `capacity` = max live entries per (layer, sequence);
 * `max_segments` = INT8 segment pool per (layer, sequence) (0 -> capacity). */
int ckv_create(const ckv_config* cfg, const ckv_shape* shape, int32_t batch, int32_t capacity,
               int32_t max_segments, const int32_t* budget_table, ckv_engine** out);
int ckv_destroy(ckv_engine* eng);
/* Empty every cache (valid_len = 0), reset the step counter to 1. */
int ckv_reset(ckv_engine* eng, void* stream);
/* Device bytes held by the engine. */
int64_t ckv_device_bytes(const ckv_engine* eng);
/* Kernels this engine has launched so far (every entry point counts its own; launches captured
 * into a CUDA graph count once, at capture). */
int64_t ckv_launch_count(const ckv_engine* eng);

/* DecodePolicy.begin_prefill (policy.py:170-171). Host-side value. */
int ckv_begin_prefill(ckv_engine* eng, int32_t prefill_len);

/* Bulk DecodePolicy.append_prefill (policy.py:165-168): appends n entries per
 * (layer, sequence) with original positions first_pos..first_pos+n-1 and
 * generation step = position - prefill_len. */
int ckv_prefill(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* k,
                const void* v, int32_t n, int32_t first_pos, void* stream);

/* tiled_attention (attention.py:60-102) for layers [layer_begin, +count) over
 * the current (pre-step) caches, split-K online softmax over the mixed
 * FP16/INT8 storage. Pure with respect to cache state; stages the
 * head-averaged attention mass for the next ckv_manage. `weights_out`
 * (optional, fp32 [count][batch][num_heads][capacity]) receives the
 * normalised attention weights the EMA will consume. */
int ckv_attend(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q,
               float* out, float* weights_out, void* stream);

/* ckv_attend, and `side` (a stream) waits for the point where the attention grids are submitted,
 * before the combine (split merge + EMA staging): work the caller then launches on `side` -- the
 * confidence pass of the same step -- runs beside the combine instead of taking SM room from the
 * attention grids. The caller joins `side` back before ckv_manage. */
int ckv_attend_fork(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q, float* out,
                    float* weights_out, void* stream, void* side);

/* ckv_attend + ckv_confidence for one step (what ckv_step runs before ckv_manage): when the
 * tcgen05 grid fills the GPU, the confidence pass is launched inline as that grid's programmatic
 * dependent (its CTAs run in the SM room beside the grid; the combine follows it), otherwise it
 * runs on `side`, forked at the start of the attention. The caller joins `side` back before
 * ckv_manage either way. */
int ckv_attend_conf(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q, float* out,
                    float* weights_out, const void* logits, int32_t dtype, int64_t ld, void* stream, void* side);

/* Parity hook: stage head-averaged mass from host-supplied attention rows
 * (update_attention_ema's input, cache.py:151-171) instead of ckv_attend.
 * rows: device fp64 [batch][num_heads][ld]. Sequence b's rows must have exactly its
 * valid_len n_b entries (cache.py:164-167): ld == n_b, or ld > n_b with a NaN at column n_b
 * of head 0 (the pad of ragged per-sequence rows). Otherwise nothing is staged for that
 * sequence and its next ckv_manage record carries the shape status (ValueError). */
int ckv_stage_rows(ckv_engine* eng, int32_t layer, const double* rows, int32_t ld, void* stream);

/* Head-sharded EMA input: `w` = the ckv_attend weights_out of every head
 * shard for layers [layer_begin, +count), all-gathered in shard order, device fp32
 * [shards][count][batch][num_heads][capacity] (num_heads = this shard's query heads).
 * Stages the head mean over all shards' heads in global head order — bit-identical to an
 * unsharded engine's. Replaces the head mean of update_attention_ema (cache.py:171). */
int ckv_stage_weights(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const float* w,
                      int32_t shards, void* stream);

/* Head-sharded EMA input as a chain in global head order (exact at
 * L*B*capacity*8 bytes per hop instead of every head's weights): shard r adds its own heads'
 * ckv_attend weights_out (`w`, fp32 [count][batch][num_heads][capacity]), in head order, to
 * shard r-1's fp64 running sums (`acc_in`, [count][batch][capacity]; NULL on shard 0) into
 * `acc_out` (may alias acc_in). The last shard's sums equal a single GPU's sequential head sum
 * bit for bit; every shard then stages mean = sum / total_heads with ckv_stage_mass
 * (update_attention_ema's head mean, cache.py:171). */
int ckv_head_partial(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const float* w, const double* acc_in,
                     double* acc_out, void* stream);
int ckv_stage_mass(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const double* acc, int32_t total_heads,
                   void* stream);

/* Vocab-sharded confidence: this engine's vocab_size is its logits slice, which starts at
 * global id `vocab_offset`. ckv_confidence_partial writes the shard's merged online-softmax
 * tuple (device fp64 [batch][8]); after an all-gather ([shards][batch][8], shard order),
 * ckv_confidence_merge finalises features, tier and arg-max over `vocab_total` ids. */
int ckv_confidence_partial(ckv_engine* eng, const void* logits, int32_t dtype, int64_t ld,
                           int64_t vocab_offset, double* partial_out, void* stream);
int ckv_confidence_merge(ckv_engine* eng, const double* partials, int32_t shards, int64_t vocab_total,
                         void* stream);

/* stable_softmax + confidence_score + select_budget + greedy sample
 * (confidence.py:31-87, policy.py:175-185) for every sequence. */
int ckv_confidence(ckv_engine* eng, const void* logits, int32_t dtype, int64_t ld, void* stream);

/* ConfKVEngine._manage + append (policy.py:199-206, 256-274) for every
 * (layer, sequence): EMA commit, budget, rank, select, compact, INT8 window,
 * append of k_new/v_new at step `step`. kept_map / kept_len optional. */
int ckv_manage(ckv_engine* eng, int32_t step, const void* k_new, const void* v_new,
               int32_t* kept_map, int32_t* kept_len, void* stream);

/* attend(all layers) + confidence + manage in one call (policy.step with the
 * attention computed inside). The confidence pass only reads the
 * logits, so it runs on an engine-owned side stream forked from / joined back
 * into `stream` (graph-capture safe) beside the attention. */
int ckv_step(ckv_engine* eng, int32_t step, const void* logits, int32_t dtype, int64_t ld,
             const void* q, const void* k_new, const void* v_new, float* out, int32_t* kept_map,
             int32_t* kept_len, void* stream);

/* Compact kept-index map: from the next ckv_manage / ckv_step on (captured into graphs at
 * capture time), K3 also writes each (layer, sequence)'s evicted pre-step storage indices,
 * ascending, to victims[layer][batch][capacity] (device int32; the first `evicted` entries of
 * the record are valid). The kept map is their complement in [0, len_pre) (policy.py:117-127,
 * cache.py:206) -- one int per cache in the steady state instead of `capacity`. NULL stops it. */
int ckv_victims_out(ckv_engine* eng, int32_t* victims);

/* Matched-rate replay (baselines.py:138-191): this step's eviction count per
 * (layer, sequence), counts[layer][batch] (host int32), and for
 * CKV_POLICY_MATCHED_RANDOM the victims' storage indices, victims[layer][batch][max_victims]
 * (host int32, the first counts[l][b] of each row used; NULL otherwise). Consumed by the
 * next ckv_manage; a count above valid_len - protected_p is reported as a ValueError
 * by the records. */
int ckv_set_victims(ckv_engine* eng, const int32_t* counts, const int32_t* victims, int32_t max_victims,
                    void* stream);

/* Decode-loop glue (no engine state): split a fused QKV projection's bf16 rows
 * qkv[batch][d + 2*kvd] = [q | k | v] into fp16 q[batch][d], k[batch][kvd], v[batch][kvd]
 * (the query input of ckv_attend and the new-entry K/V of ckv_manage). d, kvd multiples
 * of 8, pointers 16-byte aligned. Stands in for ReferenceModel.forward's per-layer
 * x @ w_q / w_k / w_v (simulator.py:79-81) feeding tiled_attention and new_kv. */
int ckv_qkv_split(const void* qkv, int32_t batch, int32_t d, int32_t kvd, void* q, void* k, void* v,
                  void* stream);

/* The greedy token of the last confidence pass for every sequence (policy.py:181-185),
 * copied device-to-device into tokens[batch] (int32) on `stream`: lets a decode loop feed
 * the next step's embedding lookup without a host round trip (simulator.py:468-476). */
int ckv_tokens(ckv_engine* eng, int32_t* tokens, void* stream);

/* Parity hook: copy the head-averaged attention mass staged for (layer, seq) by the last
 * ckv_attend / ckv_stage_rows / ckv_stage_weights (the `mean` of update_attention_ema,
 * cache.py:171; indexed by pre-step storage index, `count` = the len_pre of that step) into
 * HOST memory (synchronises). ckv_manage reads but never modifies it. */
int ckv_read_staged(ckv_engine* eng, int32_t layer, int32_t seq, int32_t count, double* mass, void* stream);

/* Host-pipeline helper (no engine state; used by the Python HostPipeline's steady state, one
 * call per decode step instead of a dozen runtime calls from Python): copy a step's packed
 * inputs H2D on `h2d` (after `ev_done`, the previous step that read this input set, unless
 * first_use), launch the step's captured graph on `compute` once the inputs landed and the
 * previous user of its output buffer was copied out (`ev_out`), then copy `out_bytes` of
 * output D2H on `d2h`. Events: ev_in = inputs landed, ev_done = step done, ev_out = output
 * copied. Streams / events / graph exec are cudaStream_t / cudaEvent_t / cudaGraphExec_t. */
int ckv_pipe_submit(void* graph_exec, void* compute, void* h2d, void* d2h, void* in_dev, const void* in_host,
                    int64_t in_bytes, void* ev_in, void* ev_done, void* ev_out, int32_t first_use, void* out_host,
                    const void* out_dev, int64_t out_bytes, void* out2_host, const void* out2_dev,
                    int64_t out2_bytes);

/* Gather the last manage's records and each cache's first `vmax` victims (victims: the
 * ckv_victims_out buffer, or NULL) into one device block `dst` of int32 words
 * [num_layers*batch][8] layer records, [batch][14] sequence records, [num_layers*batch][vmax]
 * victims -- so a pipeline copies a step's host-bound results D2H in one copy, off the step's
 * stream (capture-safe). */
int ckv_pack_outputs(ckv_engine* eng, int32_t* dst, const int32_t* victims, int32_t vmax, void* stream);

/* Copy the last step's records to HOST memory (synchronises `stream`).
 * layers: [num_layers][batch]; seqs: [batch]. Either may be NULL. */
int ckv_read_records(ckv_engine* eng, ckv_layer_record* layers, ckv_seq_record* seqs, void* stream);

/* Asynchronous ckv_read_records: enqueue the copies on `stream` and return (no
 * synchronisation; with pinned host buffers the copy overlaps later work). The
 * records are valid once `stream` has reached this point. */
int ckv_copy_records(ckv_engine* eng, ckv_layer_record* layers, ckv_seq_record* seqs, void* stream);

/* Debug/parity dump of one (layer, sequence) cache into HOST buffers
 * (synchronises). Arrays sized by capacity; segment scales are returned in
 * storage order of first use (the reference's renumbered segment ids).
 *   positions,steps int64[cap]; ema double[cap]; seen uint8[cap];
 *   segment int32[cap] (reference numbering, -1 = HIGH);
 *   keys, values float32[cap][Hkv][D] (dequantized view, like read_block);
 *   k_codes, v_codes int8[cap][Hkv][D];
 *   seg_k_scale, seg_v_scale float32[max_segments][Hkv][D]; seg_count int32[max_segments]
 * Any output pointer may be NULL (that array is not copied from the device).
 * Returns valid_len via *n_out and live segment count via *nseg_out. */
int ckv_read_cache(ckv_engine* eng, int32_t layer, int32_t seq, int32_t* n_out, int32_t* nseg_out,
                   int64_t* positions, int64_t* steps, double* ema, uint8_t* seen, int32_t* segment,
                   float* keys, float* values, int8_t* k_codes, int8_t* v_codes,
                   float* seg_k_scale, float* seg_v_scale, int32_t* seg_count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CONFKV_B200_H */
