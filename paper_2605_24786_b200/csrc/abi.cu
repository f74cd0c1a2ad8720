// C ABI (include/confkv_b200.h): engine lifetime, argument validation, launch
// sequencing and the debug/parity readers. No compute happens on the host;
// every entry point except create/destroy/read_* is asynchronous.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include <cudaTypedefs.h>

#include "ckv_internal.cuh"

namespace {

thread_local char g_err[1024] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(e == cudaErrorMemoryAllocation ? CKV_ENOMEM : CKV_ECUDA, "%s: %s", where,
              cudaGetErrorString(e));
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kDefaultLossySegments = 32;   // default max_segments (see ckv_create)

// 2-D row-gather descriptor: rows x cols elements, one-row box (gather4 loads 4 rows).
bool encode_rows(CUtensorMap* m, void* base, CUtensorMapDataType dt, uint64_t rows, uint64_t cols,
                 uint64_t elem_bytes, uint32_t box_cols = 0,
                 CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE, uint64_t row_bytes = 0) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_bytes ? row_bytes : cols * elem_bytes};
  cuuint32_t box[2] = {box_cols ? box_cols : (cuuint32_t)cols, 1};
  cuuint32_t es[2] = {1, 1};
  return fn(m, dt, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct ckv_engine {
  ckv::Dev d{};
  ckv::Maps maps{};
  ckv::Cfg c{};
  ckv_config cfg{};
  ckv_shape shape{};
  int batch = 0, cap = 0, smax = 0, nblk_conf = 0, max_budget = 0, nsm = 148;
  int tc_mode = 0;   // CKV_TC=on|off forces the persistent tcgen05 K2 grid on / off (tests, A/B)
  bool unbounded = false;   // entries were appended outside a step after stepping began
  int t_expected = 1;
  char* arena = nullptr;
  size_t bytes = 0;
  std::vector<char> attended;   // per layer, this step
  std::vector<int> pf_count;    // per layer: entries prefilled before the first step (host-side bound check)
  // ckv_step forks K1 (independent of the attention) onto a side stream so it runs beside K2
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_mid = nullptr;   // ckv_attend_fork: after the attention grids, before the combine
  int64_t launches = 0;           // kernels launched by this engine (ckv_launch_count)
};

extern "C" {

const char* ckv_last_error(void) { return g_err; }

int ckv_version(void) { return 100; }

int ckv_create(const ckv_config* cfg, const ckv_shape* shape, int32_t batch, int32_t capacity,
               int32_t max_segments, const int32_t* budget_table, ckv_engine** out) {
  if (!cfg || !shape || !budget_table || !out) return fail(CKV_EINVAL, "null argument");
  *out = nullptr;
  const ckv_shape& s = *shape;
  if (s.num_layers <= 0 || s.num_heads <= 0 || s.num_kv_heads <= 0 || s.head_dim <= 0 || s.vocab_size <= 0)
    return fail(CKV_ECONFIG, "shape fields must be strictly positive");
  if (s.num_heads % s.num_kv_heads) return fail(CKV_ECONFIG, "num_heads must be a multiple of num_kv_heads");
  if (s.vocab_size < 2) return fail(CKV_EINVAL, "need a vocabulary of at least 2 logits");
  const int G = s.num_heads / s.num_kv_heads;
  if (!ckv::attend_supported(s.head_dim, G))
    return fail(CKV_ECONFIG, "unsupported (head_dim=%d, group=%d): head_dim in {16,32,64,128}, group in {1,2,4,5,8}",
                s.head_dim, G);
  if (batch <= 0 || capacity <= 1) return fail(CKV_EINVAL, "batch must be > 0 and capacity > 1");
  if (cfg->protected_p < 0 || cfg->fp16_window_w < 0) return fail(CKV_ECONFIG, "negative window");
  if (cfg->policy < CKV_POLICY_CONFKV || cfg->policy > CKV_POLICY_MATCHED_ATTENTION)
    return fail(CKV_ECONFIG, "unknown policy %d", cfg->policy);
  if (cfg->policy != CKV_POLICY_CONFKV && cfg->quantize)
    return fail(CKV_ECONFIG, "the comparison policies never quantize (baselines.py)");
  if (cfg->policy == CKV_POLICY_SLIDING && cfg->policy_param < 1)
    return fail(CKV_EINVAL, "window must be >= 1, got %d", cfg->policy_param);
  if (cfg->policy == CKV_POLICY_HEAVY_HITTER && cfg->policy_param < cfg->protected_p)
    return fail(CKV_EINVAL, "cap %d smaller than protected window %d", cfg->policy_param, cfg->protected_p);
  if ((cfg->policy == CKV_POLICY_SLIDING || cfg->policy == CKV_POLICY_HEAVY_HITTER) &&
      cfg->policy_param + 1 > capacity)
    return fail(CKV_ECONFIG, "capacity %d must exceed the window / cap %d", capacity, cfg->policy_param);
  for (int l = 0; l < s.num_layers; ++l) {
    const int a = budget_table[2 * l], b = budget_table[2 * l + 1];
    if (a < 0 || b < 0) return fail(CKV_ECONFIG, "negative budget at layer %d", l);
    if (a + 1 > capacity || b + 1 > capacity)
      return fail(CKV_ECONFIG, "capacity %d must exceed every budget (layer %d: %d/%d)", capacity, l, a, b);
  }
  ckv_engine* e = new ckv_engine();
  e->cfg = *cfg;
  e->shape = s;
  e->batch = batch;
  e->cap = capacity;
  // lossy-segment (scale-row) pool: a bulk prefill creates one lossy segment, decode steps
  // single-entry ones (no scale rows); exhaustion is reported, never truncated
  e->smax = max_segments > 0 ? max_segments : std::min(capacity, kDefaultLossySegments);
  e->attended.assign(s.num_layers, 0);
  e->pf_count.assign(s.num_layers, 0);
  for (int l = 0; l < 2 * s.num_layers; ++l) e->max_budget = std::max(e->max_budget, (int)budget_table[l]);
  if (cfg->policy == CKV_POLICY_SLIDING || cfg->policy == CKV_POLICY_HEAVY_HITTER)
    e->max_budget = std::max(e->max_budget, (int)cfg->policy_param);
  if (cfg->policy == CKV_POLICY_FULL) e->max_budget = capacity;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&e->nsm, cudaDevAttrMultiProcessorCount, dev);
    const char* tc = getenv("CKV_TC");
    e->tc_mode = !tc ? 0 : !strcmp(tc, "on") ? 1 : !strcmp(tc, "off") ? -1 : 0;
  }
  {
    // K2 path forcing for tests / A-B runs: CKV_COMB = plain1 | plain4 | staged, CKV_DYN =
    // static | dynamic (persistent tcgen05 item schedule); unset = the launch-size rules
    const char* cb = getenv("CKV_COMB");
    e->d.comb_force = !cb ? -1 : !strcmp(cb, "plain1") ? 0 : !strcmp(cb, "plain4") ? 1 : !strcmp(cb, "staged") ? 2 : -1;
    const char* fs = getenv("CKV_FSTREAM");
    e->d.fs_force = fs ? atoi(fs) : -1;
    const char* gc = getenv("CKV_GENCAP");
    e->d.gen_cap = gc ? atoi(gc) : 1;
    const char* kt = getenv("CKV_K3T");
    e->d.k3t_force = kt ? atoi(kt) : 0;
    const char* dy = getenv("CKV_DYN");
    e->d.dyn_force = !dy ? -1 : !strcmp(dy, "static") ? 0 : !strcmp(dy, "dynamic") ? 1 : -1;
  }

  ckv::Dev& d = e->d;
  d.L = s.num_layers; d.B = batch; d.Hq = s.num_heads; d.Hkv = s.num_kv_heads; d.D = s.head_dim;
  d.V = s.vocab_size; d.G = G; d.cap = capacity; d.smax = e->smax; d.C = d.L * d.B;
  d.nsid = e->smax + capacity;
  d.nsplit = (capacity + ckv::kSplitTokens - 1) / ckv::kSplitTokens;
  d.npart = 2 * d.nsplit;
  d.sld = (capacity + 63) / 64 * 64;
  d.quant = cfg->quantize ? 1 : 0;
  // K3's staged fast path (one metadata read per step) for caches up to 4,352 entries;
  // CKV_K3_STAGE=0 turns it off (A/B)
  d.kstage = (getenv("CKV_K3_STAGE") && atoi(getenv("CKV_K3_STAGE")) == 0) ? 0 : std::min(capacity, 4352);
  e->nblk_conf = (d.V + ckv::kConfPerBlock - 1) / ckv::kConfPerBlock;

  const size_t C = d.C, cap = capacity, row = (size_t)d.Hkv * d.D, sm = e->smax, ns = d.nsid;
  struct Item { void** p; size_t bytes; };
  std::vector<Item> items = {
      {(void**)&d.kf, C * cap * row * 2}, {(void**)&d.vf, C * cap * row * 2},
      {(void**)&d.slot, C * cap * 4}, {(void**)&d.pos, C * cap * 4}, {(void**)&d.stp, C * cap * 4},
      {(void**)&d.ema, C * cap * 8}, {(void**)&d.seen, C * cap}, {(void**)&d.seg, C * cap * 4},
      {(void**)&d.len, C * 4}, {(void**)&d.n8, C * 4}, {(void**)&d.nq, C * 4}, {(void**)&d.fstk, C * cap * 4},
      {(void**)&d.ftop, C * 4}, {(void**)&d.ksc, C * sm * row * 4}, {(void**)&d.vsc, C * sm * row * 4},
      {(void**)&d.scnt, C * ns * 4}, {(void**)&d.sstk, C * ns * 4}, {(void**)&d.stop, C * 4},
      {(void**)&d.stopb, C * 4}, {(void**)&d.clo, C * 4}, {(void**)&d.ccnt, C * 4},
      {(void**)&d.socc, C * cap * 4}, {(void**)&d.vslot, C * cap * 4},
      {(void**)&d.nseg, C * 4}, {(void**)&d.score, C * d.Hq * (size_t)d.sld * 4},
      {(void**)&d.pm, C * d.Hq * d.npart * 4}, {(void**)&d.pz, C * d.Hq * d.npart * 4},
      {(void**)&d.po, C * d.Hq * d.npart * d.D * 4}, {(void**)&d.abar, C * cap * 8},
      {(void**)&d.att_len, C * 4}, {(void**)&d.cpart, (size_t)batch * e->nblk_conf * 8 * 8},
      {(void**)&d.ticket, (size_t)batch * 4}, {(void**)&d.k1exit, 4}, {(void**)&d.conf, (size_t)batch * sizeof(ckv_seq_record)},
      {(void**)&d.keys, C * cap * 8}, {(void**)&d.vseg, C * cap * 4}, {(void**)&d.qlo, C * 4},
      {(void**)&d.qcnt, C * 4}, {(void**)&d.qseg, C * 4}, {(void**)&d.newslot, C * 4},
      {(void**)&d.pf_base, C * 4}, {(void**)&d.pf_status, C * 4}, {(void**)&d.rec, C * sizeof(ckv_layer_record)},
      {(void**)&d.budget, (size_t)d.L * 2 * 4}, {(void**)&d.tnext, 4},
      {(void**)&d.evcnt, C * 4}, {(void**)&d.work, 4},
      {(void**)&d.vlist, cfg->policy == CKV_POLICY_MATCHED_RANDOM ? C * cap * 4 : 4},
  };
  size_t total = 0;
  for (auto& it : items) total += align_up(it.bytes);
  cudaError_t err = cudaMalloc((void**)&e->arena, total);
  if (err != cudaSuccess) {
    delete e;
    return cuda_fail(err, "ckv_create: cudaMalloc");
  }
  e->bytes = total;
  size_t off = 0;
  for (auto& it : items) { *it.p = e->arena + off; off += align_up(it.bytes); }
  // INT8 codes of lossy entries live in the fp16 slot pool, two code rows per slot head row
  d.kq = reinterpret_cast<int8_t*>(d.kf);
  d.vq = reinterpret_cast<int8_t*>(d.vf);
  cudaMemset(e->arena, 0, total);
  cudaMemcpy(d.budget, budget_table, (size_t)d.L * 2 * 4, cudaMemcpyHostToDevice);
  cudaMemset(d.conf, 0, (size_t)batch * sizeof(ckv_seq_record));

  ckv::Cfg& c = e->c;
  c.tau = cfg->tau; c.alpha = cfg->alpha; c.one_m_alpha = 1.0 - cfg->alpha;
  c.lam = cfg->ema_lambda; c.one_m_lam = 1.0 - cfg->ema_lambda;
  c.wH = cfg->w_entropy; c.wM = cfg->w_margin; c.wP = cfg->w_top;
  c.temperature = cfg->temperature; c.P = cfg->protected_p; c.W = cfg->fp16_window_w;
  c.quantize = cfg->quantize; c.temp_mode = cfg->temperature_mode; c.prefill_len = 0;
  c.policy = cfg->policy; c.param = cfg->policy_param;
  if (c.policy == CKV_POLICY_MATCHED_RECENCY || c.policy == CKV_POLICY_MATCHED_ATTENTION) {
    // select_victims(cache, count, protected, alpha) with alpha = 0 / 1 (baselines.py:170-172)
    c.alpha = c.policy == CKV_POLICY_MATCHED_ATTENTION ? 1.0 : 0.0;
    c.one_m_alpha = 1.0 - c.alpha;
  }

  {
    const uint64_t rows = (uint64_t)C * cap * d.Hkv;
    bool ok = encode_rows(&e->maps.kf, d.kf, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, d.D, 2) &&
              encode_rows(&e->maps.vf, d.vf, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, d.D, 2) &&
              encode_rows(&e->maps.kq, d.kq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2 * rows, d.D, 1) &&
              encode_rows(&e->maps.vq, d.vq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2 * rows, d.D, 1);
    if (ok && d.D >= 64) {
      const auto SW = CU_TENSOR_MAP_SWIZZLE_128B;
      ok = encode_rows(&e->maps.kf_sw, d.kf, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, d.D, 2, 64, SW) &&
           encode_rows(&e->maps.vf_sw, d.vf, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rows, d.D, 2, 64, SW) &&
           encode_rows(&e->maps.kq_sw, d.kq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2 * rows, d.D, 1, d.D, SW) &&
           encode_rows(&e->maps.vq_sw, d.vq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2 * rows, d.D, 1, d.D, SW);
    }
    if (!ok) {
      cudaFree(e->arena);
      delete e;
      return fail(CKV_ECUDA, "ckv_create: cuTensorMapEncodeTiled failed");
    }
  }
  err = ckv::launch_init(d, 0);
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    cudaFree(e->arena);
    delete e;
    return cuda_fail(err, "ckv_create: init");
  }
  *out = e;
  return CKV_OK;
}

int ckv_destroy(ckv_engine* eng) {
  if (!eng) return CKV_OK;
  if (eng->ev_fork) cudaEventDestroy(eng->ev_fork);
  if (eng->ev_join) cudaEventDestroy(eng->ev_join);
  if (eng->ev_mid) cudaEventDestroy(eng->ev_mid);
  if (eng->side) cudaStreamDestroy(eng->side);
  cudaFree(eng->arena);
  delete eng;
  return CKV_OK;
}

int64_t ckv_device_bytes(const ckv_engine* eng) { return eng ? (int64_t)eng->bytes : 0; }

int64_t ckv_launch_count(const ckv_engine* eng) { return eng ? eng->launches : 0; }

int ckv_reset(ckv_engine* eng, void* stream) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  cudaError_t e = ckv::launch_init(eng->d, (cudaStream_t)stream);
  eng->launches += 1;
  if (e != cudaSuccess) return cuda_fail(e, "ckv_reset");
  eng->t_expected = 1;
  eng->unbounded = false;
  std::fill(eng->attended.begin(), eng->attended.end(), 0);
  std::fill(eng->pf_count.begin(), eng->pf_count.end(), 0);
  return CKV_OK;
}

int ckv_begin_prefill(ckv_engine* eng, int32_t prefill_len) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  eng->c.prefill_len = prefill_len;
  return CKV_OK;
}

int ckv_prefill(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* k,
                const void* v, int32_t n, int32_t first_pos, void* stream) {
  if (!eng || !k || !v) return fail(CKV_EINVAL, "null argument");
  if (layer_begin < 0 || layer_count <= 0 || layer_begin + layer_count > eng->d.L)
    return fail(CKV_EINVAL, "layer range [%d, %d) outside [0, %d)", layer_begin, layer_begin + layer_count, eng->d.L);
  if (n <= 0) return CKV_OK;
  if (n > eng->cap) return fail(CKV_EINVAL, "prefill of %d entries exceeds capacity %d", n, eng->cap);
  if (eng->t_expected <= 1) {
    // before the first step every cache holds exactly what was prefilled: refuse a chunk that
    // would not fit (after stepping began the device checks, see pf_status)
    for (int l = layer_begin; l < layer_begin + layer_count; ++l)
      if (eng->pf_count[l] + n > eng->cap)
        return fail(CKV_EINVAL, "prefill of layer %d would hold %d entries > capacity %d (pass a larger capacity)",
                    l, eng->pf_count[l] + n, eng->cap);
    for (int l = layer_begin; l < layer_begin + layer_count; ++l) eng->pf_count[l] += n;
  }
  if (eng->t_expected > 1) eng->unbounded = true;   // lengths no longer bounded by the budgets
  if ((reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v)) % 16)
    return fail(CKV_EINVAL, "prefill K/V must be 16-byte aligned");
  cudaError_t e = ckv::launch_prefill(eng->d, eng->c, layer_begin * eng->d.B, layer_count * eng->d.B,
                                      (const __half*)k, (const __half*)v, n, first_pos, (cudaStream_t)stream);
  eng->launches += 2;
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_prefill");
}

static int attend_impl(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q, float* out,
                       float* weights_out, void* stream, cudaEvent_t mid, ckv::K1Inline* k1 = nullptr);

int ckv_attend(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q,
               float* out, float* weights_out, void* stream) {
  return attend_impl(eng, layer_begin, layer_count, q, out, weights_out, stream, nullptr);
}

int ckv_attend_fork(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q, float* out,
                    float* weights_out, void* stream, void* side) {
  if (!eng || !side) return fail(CKV_EINVAL, "null argument");
  if (!eng->ev_mid) {
    cudaError_t e = cudaEventCreateWithFlags(&eng->ev_mid, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "ckv_attend_fork: event");
  }
  int r = attend_impl(eng, layer_begin, layer_count, q, out, weights_out, stream, eng->ev_mid);
  if (r != CKV_OK) return r;
  cudaError_t e = cudaStreamWaitEvent((cudaStream_t)side, eng->ev_mid, 0);
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_attend_fork: fork");
}

int ckv_attend_conf(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q, float* out,
                    float* weights_out, const void* logits, int32_t dtype, int64_t ld, void* stream, void* side) {
  if (!eng || !logits || !side) return fail(CKV_EINVAL, "null argument");
  if (dtype != CKV_DTYPE_F32 && dtype != CKV_DTYPE_BF16 && dtype != CKV_DTYPE_F64)
    return fail(CKV_EINVAL, "unknown logits dtype %d", dtype);
  if (ld < eng->d.V) return fail(CKV_EINVAL, "ld %lld < vocab_size %d", (long long)ld, eng->d.V);
  if (!eng->ev_mid) {
    cudaError_t e = cudaEventCreateWithFlags(&eng->ev_mid, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "ckv_attend_conf: event");
  }
  // K1 inline when the tcgen05 grid fills the GPU (launch_attend decides); otherwise K1 is
  // forked onto `side` at the start of the attention
  cudaError_t e = cudaEventRecord(eng->ev_mid, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "ckv_attend_conf: fork");
  ckv::K1Inline k1{&eng->c, logits, dtype, ld, 0};
  int r = attend_impl(eng, layer_begin, layer_count, q, out, weights_out, stream, nullptr, &k1);
  if (r != CKV_OK) return r;
  // `side` always forks from the step's stream (an empty branch when K1 ran inline), so the
  // caller's join is well-formed inside a stream capture too
  e = cudaStreamWaitEvent((cudaStream_t)side, eng->ev_mid, 0);
  if (e != cudaSuccess) return cuda_fail(e, "ckv_attend_conf: fork");
  if (k1.inlined) {
    eng->launches += 1;
    return CKV_OK;
  }
  return ckv_confidence(eng, logits, dtype, ld, side);
}

static int attend_impl(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const void* q, float* out,
                       float* weights_out, void* stream, cudaEvent_t mid, ckv::K1Inline* k1) {
  if (!eng || !q) return fail(CKV_EINVAL, "null argument");
  if (layer_begin < 0 || layer_count <= 0 || layer_begin + layer_count > eng->d.L)
    return fail(CKV_EINVAL, "layer range [%d, %d) outside [0, %d)", layer_begin, layer_begin + layer_count, eng->d.L);
  if (reinterpret_cast<uintptr_t>(q) % 16) return fail(CKV_EINVAL, "q must be 16-byte aligned");
  // Width of the general-split launch: single-segment INT8 splits lie below the codes prefix,
  // which is at most the first demotion after the prefill (prefill_len - W + 1 entries) and only
  // shrinks under eviction; the kernel loops if a cache has more general splits than this.
  // Before the first step nothing is INT8 yet, so every split is general.
  // The persistent tcgen05 grid pays off from ~one 512-entry codes split per SM (NIAH decode at
  // batch 1 after the 32K -> 512 selection: 256 items, 63 -> 59 us/step with it); smaller
  // launches run every split on the general kernel's integer path.
  {
    const int nq_est = eng->c.quantize ? std::max(0, std::min(eng->c.prefill_len - eng->c.W + 1, eng->max_budget + 1))
                                       : 0;
    eng->d.gen_splits = eng->t_expected <= 1 ? eng->d.nsplit
                                             : std::max(1, eng->d.nsplit - nq_est / ckv::kSplitTokens);
    const long tc_items = (long)layer_count * eng->d.B * eng->d.Hkv * (nq_est / ckv::kSplitTokens);
    eng->d.use_tc = eng->tc_mode == 1 || (eng->tc_mode == 0 && eng->t_expected > 1 && tc_items >= eng->nsm);
    // after the first step a cache holds at most its budget + the appended entry (before it,
    // whatever was prefilled): launch widths follow that, not the capacity
    const bool bounded = eng->t_expected > 1 && !eng->unbounded && eng->c.policy != CKV_POLICY_FULL &&
                         eng->c.policy < CKV_POLICY_MATCHED_RANDOM;
    const int live = bounded ? std::min(eng->cap, eng->max_budget + 1) : eng->cap;
    eng->d.live_splits = (live + ckv::kSplitTokens - 1) / ckv::kSplitTokens;
    // general (non-codes) entries per cache ~ live - nq_est: one CTA per 512 of them (the
    // bulk steady state's FP16 window + a straddled split boundary -> one CTA per pair)
    if (eng->t_expected > 1)
      eng->d.gen_splits = std::max(1, (live - nq_est + ckv::kSplitTokens - 1) / ckv::kSplitTokens);
    eng->d.gen_splits = std::min(eng->d.gen_splits, eng->d.live_splits);
  }
  cudaError_t e = ckv::launch_attend(eng->d, eng->maps, layer_begin * eng->d.B, layer_count * eng->d.B,
                                     (const __half*)q, out, weights_out, (cudaStream_t)stream, mid, k1);
  eng->launches += ckv::last_attend_launches() - (k1 && k1->inlined ? 1 : 0);   // K1 counted by the caller
  if (e != cudaSuccess) return cuda_fail(e, "ckv_attend");
  for (int l = layer_begin; l < layer_begin + layer_count; ++l) eng->attended[l] = 1;
  return CKV_OK;
}

int ckv_stage_rows(ckv_engine* eng, int32_t layer, const double* rows, int32_t ld, void* stream) {
  if (!eng || !rows) return fail(CKV_EINVAL, "null argument");
  if (layer < 0 || layer >= eng->d.L) return fail(CKV_EINVAL, "layer %d outside [0, %d)", layer, eng->d.L);
  cudaError_t e = ckv::launch_stage_rows(eng->d, layer, rows, ld, (cudaStream_t)stream);
  eng->launches += 1;
  if (e != cudaSuccess) return cuda_fail(e, "ckv_stage_rows");
  eng->attended[layer] = 1;
  return CKV_OK;
}

int ckv_stage_weights(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const float* w,
                      int32_t shards, void* stream) {
  if (!eng || !w) return fail(CKV_EINVAL, "null argument");
  if (layer_begin < 0 || layer_count <= 0 || layer_begin + layer_count > eng->d.L)
    return fail(CKV_EINVAL, "layer range [%d, %d) outside [0, %d)", layer_begin, layer_begin + layer_count, eng->d.L);
  if (shards <= 0) return fail(CKV_EINVAL, "shards must be positive");
  cudaError_t e = ckv::launch_stage_weights(eng->d, layer_begin * eng->d.B, layer_count * eng->d.B, w, shards,
                                            (cudaStream_t)stream);
  eng->launches += 1;
  if (e != cudaSuccess) return cuda_fail(e, "ckv_stage_weights");
  for (int l = layer_begin; l < layer_begin + layer_count; ++l) eng->attended[l] = 1;
  return CKV_OK;
}

int ckv_head_partial(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const float* w, const double* acc_in,
                     double* acc_out, void* stream) {
  if (!eng || !w || !acc_out) return fail(CKV_EINVAL, "null argument");
  if (layer_begin < 0 || layer_count <= 0 || layer_begin + layer_count > eng->d.L)
    return fail(CKV_EINVAL, "layer range [%d, %d) outside [0, %d)", layer_begin, layer_begin + layer_count, eng->d.L);
  cudaError_t e = ckv::launch_head_partial(eng->d, layer_begin * eng->d.B, layer_count * eng->d.B, w, acc_in, acc_out,
                                           (cudaStream_t)stream);
  eng->launches += 1;
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_head_partial");
}

int ckv_stage_mass(ckv_engine* eng, int32_t layer_begin, int32_t layer_count, const double* acc, int32_t total_heads,
                   void* stream) {
  if (!eng || !acc) return fail(CKV_EINVAL, "null argument");
  if (layer_begin < 0 || layer_count <= 0 || layer_begin + layer_count > eng->d.L)
    return fail(CKV_EINVAL, "layer range [%d, %d) outside [0, %d)", layer_begin, layer_begin + layer_count, eng->d.L);
  if (total_heads <= 0) return fail(CKV_EINVAL, "total_heads must be positive");
  cudaError_t e = ckv::launch_stage_mass(eng->d, layer_begin * eng->d.B, layer_count * eng->d.B, acc, total_heads,
                                         (cudaStream_t)stream);
  eng->launches += 1;
  if (e != cudaSuccess) return cuda_fail(e, "ckv_stage_mass");
  for (int l = layer_begin; l < layer_begin + layer_count; ++l) eng->attended[l] = 1;
  return CKV_OK;
}

int ckv_confidence_partial(ckv_engine* eng, const void* logits, int32_t dtype, int64_t ld, int64_t vocab_offset,
                           double* partial_out, void* stream) {
  if (!eng || !logits || !partial_out) return fail(CKV_EINVAL, "null argument");
  if (dtype != CKV_DTYPE_F32 && dtype != CKV_DTYPE_BF16 && dtype != CKV_DTYPE_F64)
    return fail(CKV_EINVAL, "unknown logits dtype %d", dtype);
  if (ld < eng->d.V) return fail(CKV_EINVAL, "ld %lld < vocab slice %d", (long long)ld, eng->d.V);
  if (vocab_offset < 0 || vocab_offset > 0x7fffffff - eng->d.V) return fail(CKV_EINVAL, "bad vocab_offset");
  cudaError_t e = ckv::launch_confidence(eng->d, eng->c, logits, dtype, ld, (cudaStream_t)stream,
                                         (int)vocab_offset, partial_out);
  eng->launches += 1;
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_confidence_partial");
}

int ckv_confidence_merge(ckv_engine* eng, const double* partials, int32_t shards, int64_t vocab_total,
                         void* stream) {
  if (!eng || !partials) return fail(CKV_EINVAL, "null argument");
  if (shards <= 0 || vocab_total < 2) return fail(CKV_EINVAL, "bad shards / vocab_total");
  cudaError_t e = ckv::launch_confidence_merge(eng->d, eng->c, partials, shards, vocab_total, (cudaStream_t)stream);
  eng->launches += 1;
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_confidence_merge");
}

int ckv_confidence(ckv_engine* eng, const void* logits, int32_t dtype, int64_t ld, void* stream) {
  if (!eng || !logits) return fail(CKV_EINVAL, "null argument");
  if (dtype != CKV_DTYPE_F32 && dtype != CKV_DTYPE_BF16 && dtype != CKV_DTYPE_F64)
    return fail(CKV_EINVAL, "unknown logits dtype %d", dtype);
  if (ld < eng->d.V) return fail(CKV_EINVAL, "ld %lld < vocab_size %d", (long long)ld, eng->d.V);
  cudaError_t e = ckv::launch_confidence(eng->d, eng->c, logits, dtype, ld, (cudaStream_t)stream);
  eng->launches += 1;
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_confidence");
}

int ckv_manage(ckv_engine* eng, int32_t step, const void* k_new, const void* v_new, int32_t* kept_map,
               int32_t* kept_len, void* stream) {
  if (!eng || !k_new || !v_new) return fail(CKV_EINVAL, "null argument");
  for (int l = 0; l < eng->d.L; ++l)
    if (!eng->attended[l])
      return fail(CKV_ERUNTIME, "attention rows missing for layer %d (attend every layer before the step)", l);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (step != eng->t_expected) {
    e = ckv::launch_set_step(eng->d, step, s);
    eng->launches += 1;
  }
  if (e == cudaSuccess)
    e = ckv::launch_manage(eng->d, eng->c, (const __half*)k_new, (const __half*)v_new, kept_map, kept_len, s);
  eng->launches += 2;   // K3 + K4
  if (e != cudaSuccess) return cuda_fail(e, "ckv_manage");
  eng->t_expected = step + 1;
  std::fill(eng->attended.begin(), eng->attended.end(), 0);
  return CKV_OK;
}

int ckv_step(ckv_engine* eng, int32_t step, const void* logits, int32_t dtype, int64_t ld, const void* q,
             const void* k_new, const void* v_new, float* out, int32_t* kept_map, int32_t* kept_len,
             void* stream) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  cudaStream_t s = (cudaStream_t)stream;
  if (!eng->side) {
    cudaError_t e = cudaStreamCreateWithFlags(&eng->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&eng->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&eng->ev_join, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "ckv_step: side stream");
  }
  // K1 reads only the logits: inline beside the tcgen05 grid when that grid fills the GPU (a
  // forked K1 there took the SM slots the grid's CTAs needed -- they started up to 20 us late and
  // ended ragged -- and forked after the grids it ran past the combine), else on the side stream
  // beside the attention (ckv_attend_conf).
  int r = ckv_attend_conf(eng, 0, eng->d.L, q, out, nullptr, logits, dtype, ld, stream, eng->side);
  // join (also on failure, so the side stream never dangles in a capture)
  if (r != CKV_OK) {   // keep the side stream joined to the step's stream
    cudaEventRecord(eng->ev_fork, s);
    cudaStreamWaitEvent(eng->side, eng->ev_fork, 0);
  }
  cudaError_t e = cudaEventRecord(eng->ev_join, eng->side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, eng->ev_join, 0);
  if (r != CKV_OK) return r;
  if (e != cudaSuccess) return cuda_fail(e, "ckv_step: join");
  return ckv_manage(eng, step, k_new, v_new, kept_map, kept_len, stream);
}

int ckv_victims_out(ckv_engine* eng, int32_t* victims) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  eng->d.victims = victims;
  return CKV_OK;
}

int ckv_set_victims(ckv_engine* eng, const int32_t* counts, const int32_t* victims, int32_t max_victims,
                    void* stream) {
  if (!eng || !counts) return fail(CKV_EINVAL, "null argument");
  const int pol = eng->c.policy;
  if (pol < CKV_POLICY_MATCHED_RANDOM) return fail(CKV_ERUNTIME, "ckv_set_victims needs a matched-rate policy");
  cudaStream_t s = (cudaStream_t)stream;
  const int C = eng->d.C;
  cudaError_t e = cudaMemcpyAsync(eng->d.evcnt, counts, (size_t)C * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && pol == CKV_POLICY_MATCHED_RANDOM) {
    if (!victims || max_victims < 0 || max_victims > eng->cap)
      return fail(CKV_EINVAL, "random mode needs victims[layers][batch][max_victims <= capacity]");
    if (max_victims > 0)
      e = cudaMemcpy2DAsync(eng->d.vlist, (size_t)eng->cap * 4, victims, (size_t)max_victims * 4,
                            (size_t)max_victims * 4, (size_t)C, cudaMemcpyHostToDevice, s);
  }
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_set_victims");
}

int ckv_tokens(ckv_engine* eng, int32_t* tokens, void* stream) {
  if (!eng || !tokens) return fail(CKV_EINVAL, "null argument");
  // strided device-to-device gather of each sequence record's token (graph-capturable)
  cudaError_t e = cudaMemcpy2DAsync(tokens, sizeof(int32_t),
                                    reinterpret_cast<const char*>(eng->d.conf) + offsetof(ckv_seq_record, token),
                                    sizeof(ckv_seq_record), sizeof(int32_t), (size_t)eng->d.B,
                                    cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_tokens");
}

int ckv_pipe_submit(void* graph_exec, void* compute, void* h2d, void* d2h, void* in_dev, const void* in_host,
                    int64_t in_bytes, void* ev_in, void* ev_done, void* ev_out, int32_t first_use, void* out_host,
                    const void* out_dev, int64_t out_bytes, void* out2_host, const void* out2_dev,
                    int64_t out2_bytes) {
  // (a null stream is the legacy default stream)
  if (!graph_exec || !ev_in || !ev_done || !ev_out) return fail(CKV_EINVAL, "null argument");
  cudaStream_t sc = (cudaStream_t)compute, si = (cudaStream_t)h2d, so = (cudaStream_t)d2h;
  cudaEvent_t ei = (cudaEvent_t)ev_in, ed = (cudaEvent_t)ev_done, eo = (cudaEvent_t)ev_out;
  cudaError_t e = cudaSuccess;
  // inputs: once the step that last read this input set is done
  if (!first_use) e = cudaStreamWaitEvent(si, ed, 0);
  if (e == cudaSuccess && in_bytes > 0) e = cudaMemcpyAsync(in_dev, in_host, (size_t)in_bytes, cudaMemcpyHostToDevice, si);
  if (e == cudaSuccess) e = cudaEventRecord(ei, si);
  // the step: after its inputs landed and the previous user of its output buffer was copied out
  if (e == cudaSuccess) e = cudaStreamWaitEvent(sc, ei, 0);
  if (e == cudaSuccess && !first_use) e = cudaStreamWaitEvent(sc, eo, 0);
  if (e == cudaSuccess) e = cudaGraphLaunch((cudaGraphExec_t)graph_exec, sc);
  if (e == cudaSuccess) e = cudaEventRecord(ed, sc);
  // output
  if (e == cudaSuccess) e = cudaStreamWaitEvent(so, ed, 0);
  if (e == cudaSuccess && out_host && out_bytes > 0)
    e = cudaMemcpyAsync(out_host, out_dev, (size_t)out_bytes, cudaMemcpyDeviceToHost, so);
  if (e == cudaSuccess && out2_host && out2_bytes > 0)
    e = cudaMemcpyAsync(out2_host, out2_dev, (size_t)out2_bytes, cudaMemcpyDeviceToHost, so);
  if (e == cudaSuccess) e = cudaEventRecord(eo, so);
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_pipe_submit");
}

int ckv_read_records(ckv_engine* eng, ckv_layer_record* layers, ckv_seq_record* seqs, void* stream) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (layers) e = cudaMemcpyAsync(layers, eng->d.rec, (size_t)eng->d.C * sizeof(ckv_layer_record), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && seqs)
    e = cudaMemcpyAsync(seqs, eng->d.conf, (size_t)eng->d.B * sizeof(ckv_seq_record), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_read_records");
}

namespace {
// One step's host-bound outputs gathered into one contiguous device block (one D2H copy):
// [C][8] layer-record words, [B][14] sequence-record words, [C][vmax] leading victims.
__global__ void pack_outputs(const int32_t* __restrict__ rec, const int32_t* __restrict__ conf,
                             const int32_t* __restrict__ victims, int C, int B, int cap, int vmax,
                             int32_t* __restrict__ dst) {
  const int nr = C * 8, ns = B * 14, nv = victims ? C * vmax : 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nr + ns + nv; i += gridDim.x * blockDim.x) {
    if (i < nr) dst[i] = rec[i];
    else if (i < nr + ns) dst[i] = conf[i - nr];
    else {
      const int k = i - nr - ns, c = k / vmax;
      dst[i] = victims[(size_t)c * cap + (k - c * vmax)];
    }
  }
}
}  // namespace

int ckv_pack_outputs(ckv_engine* eng, int32_t* dst, const int32_t* victims, int32_t vmax, void* stream) {
  if (!eng || !dst || vmax < 0) return fail(CKV_EINVAL, "bad argument");
  static_assert(sizeof(ckv_layer_record) == 32 && sizeof(ckv_seq_record) == 56, "record words");
  const ckv::Dev& d = eng->d;
  const int total = d.C * 8 + d.B * 14 + (victims ? d.C * vmax : 0);
  pack_outputs<<<(total + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const int32_t*>(d.rec), reinterpret_cast<const int32_t*>(d.conf), victims, d.C, d.B, d.cap,
      vmax, dst);
  eng->launches += 1;
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_pack_outputs");
}

int ckv_copy_records(ckv_engine* eng, ckv_layer_record* layers, ckv_seq_record* seqs, void* stream) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaSuccess;
  if (layers) e = cudaMemcpyAsync(layers, eng->d.rec, (size_t)eng->d.C * sizeof(ckv_layer_record), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && seqs)
    e = cudaMemcpyAsync(seqs, eng->d.conf, (size_t)eng->d.B * sizeof(ckv_seq_record), cudaMemcpyDeviceToHost, s);
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_copy_records");
}

int ckv_read_cache(ckv_engine* eng, int32_t layer, int32_t seq, int32_t* n_out, int32_t* nseg_out,
                   int64_t* positions, int64_t* steps, double* ema, uint8_t* seen, int32_t* segment,
                   float* keys, float* values, int8_t* k_codes, int8_t* v_codes, float* seg_k_scale,
                   float* seg_v_scale, int32_t* seg_count, void* stream) {
  if (!eng) return fail(CKV_EINVAL, "null engine");
  const ckv::Dev& d = eng->d;
  if (layer < 0 || layer >= d.L || seq < 0 || seq >= d.B) return fail(CKV_EINVAL, "bad (layer, seq)");
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "ckv_read_cache sync");
  const int c = layer * d.B + seq;
  const size_t cap = d.cap, row = (size_t)d.Hkv * d.D, base = (size_t)c * cap;
  int n = 0, n8 = 0, nseg = 0;
  cudaMemcpy(&n, d.len + c, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&n8, d.n8 + c, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&nseg, d.nseg + c, 4, cudaMemcpyDeviceToHost);
  std::vector<int32_t> slot(cap), pos(cap), stp(cap), sg(cap);
  std::vector<double> em(cap);
  std::vector<uint8_t> sn(cap);
  const bool want_kv = keys || values || k_codes || v_codes;
  const bool want_seg = want_kv || segment || seg_k_scale || seg_v_scale || seg_count;
  const bool want_rows = want_kv || seg_k_scale || seg_v_scale;
  if (want_rows) cudaMemcpy(slot.data(), d.slot + base, cap * 4, cudaMemcpyDeviceToHost);
  if (positions) cudaMemcpy(pos.data(), d.pos + base, cap * 4, cudaMemcpyDeviceToHost);
  if (steps) cudaMemcpy(stp.data(), d.stp + base, cap * 4, cudaMemcpyDeviceToHost);
  if (want_seg) cudaMemcpy(sg.data(), d.seg + base, cap * 4, cudaMemcpyDeviceToHost);
  if (ema) cudaMemcpy(em.data(), d.ema + base, cap * 8, cudaMemcpyDeviceToHost);
  if (seen) cudaMemcpy(sn.data(), d.seen + base, cap, cudaMemcpyDeviceToHost);
  std::vector<__half> kf, vf;
  if (want_rows) {
    kf.resize(cap * row); vf.resize(cap * row);
    cudaMemcpy(kf.data(), d.kf + base * row, cap * row * 2, cudaMemcpyDeviceToHost);
    cudaMemcpy(vf.data(), d.vf + base * row, cap * row * 2, cudaMemcpyDeviceToHost);
  }
  const size_t sm = d.smax, ns = d.nsid;
  std::vector<float> ks, vs;
  std::vector<int32_t> sc(ns);
  if (want_kv || seg_k_scale || seg_v_scale) {
    ks.resize(sm * row); vs.resize(sm * row);
    cudaMemcpy(ks.data(), d.ksc + (size_t)c * sm * row, sm * row * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(vs.data(), d.vsc + (size_t)c * sm * row, sm * row * 4, cudaMemcpyDeviceToHost);
  }
  if (seg_count) cudaMemcpy(sc.data(), d.scnt + (size_t)c * ns, ns * 4, cudaMemcpyDeviceToHost);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "ckv_read_cache copy");
  // codes of a lossy entry: its code row (code slot cs = 2*slot + half); a single-entry segment
  // (id >= smax) keeps its fp16 row, its code and scale are quantize_segment of that one row
  // (quantizer.py:28-33: scale = |x|/127, code = copysign(floor(|x/scale| + 0.5)), clipped)
  const int D = d.D;
  auto lossy_code = [&](const std::vector<__half>& h, int cs, size_t r) {
    const size_t hh = r / D, dd = r % D;   // the code row of head hh within this cache's bytes
    const size_t crow = ((size_t)(cs >> 1) * d.Hkv + hh) * 2 + (cs & 1);
    return reinterpret_cast<const int8_t*>(h.data())[crow * D + dd];
  };
  auto single = [](float x, float* scale_out) -> int8_t {
    const float scale = std::fabs(x) / 127.0f;
    if (scale_out) *scale_out = scale;
    if (!(scale > 0.f)) return 0;
    const float s = x / scale;
    float code = std::copysign(std::floor(std::fabs(s) + 0.5f), s);
    code = std::fmin(std::fmax(code, -127.f), 127.f);
    return (int8_t)(int)code;
  };

  // reference numbering of segments: order of first appearance in storage order
  std::map<int, int> canon;
  std::vector<int> order;
  for (int i = 0; i < n; ++i)
    if (want_seg && sg[i] >= 0 && !canon.count(sg[i])) { canon[sg[i]] = (int)order.size(); order.push_back(sg[i]); }
  if (n_out) *n_out = n;
  if (nseg_out) *nseg_out = nseg;
  for (int i = 0; i < n; ++i) {
    if (positions) positions[i] = pos[i];
    if (steps) steps[i] = stp[i];
    if (ema) ema[i] = em[i];
    if (seen) seen[i] = sn[i];
    const bool q8 = want_seg && sg[i] >= 0;
    if (segment) segment[i] = q8 ? canon[sg[i]] : -1;
    if (!want_kv) continue;
    const bool lossy = q8 && sg[i] < (int)sm;   // codes form: slot[i] is a code slot
    const size_t src = lossy ? 0 : (size_t)slot[i] * row;
    for (size_t r = 0; r < row; ++r) {
      const size_t dst = (size_t)i * row + r;
      const float xk = lossy ? 0.f : __half2float(kf[src + r]), xv = lossy ? 0.f : __half2float(vf[src + r]);
      int8_t ck = 0, cv = 0;
      float sk = 0.f, sv = 0.f;
      if (lossy) {
        ck = lossy_code(kf, slot[i], r);
        cv = lossy_code(vf, slot[i], r);
        const size_t so = (size_t)sg[i] * row + r;
        sk = ks[so];
        sv = vs[so];
      } else if (q8) {
        ck = single(xk, &sk);
        cv = single(xv, &sv);
      }
      if (k_codes) k_codes[dst] = ck;
      if (v_codes) v_codes[dst] = cv;
      if (q8) {   // dequantised view, as read_block (cache.py:247-251, quantizer.py:37-39)
        if (keys) keys[dst] = (float)ck * sk;
        if (values) values[dst] = (float)cv * sv;
      } else {
        if (keys) keys[dst] = xk;
        if (values) values[dst] = xv;
      }
    }
  }
  for (size_t k = 0; k < order.size(); ++k) {
    const int id = order[k];
    if (id < (int)sm) {
      const size_t so = (size_t)id * row;
      if (seg_k_scale) memcpy(seg_k_scale + k * row, ks.data() + so, row * 4);
      if (seg_v_scale) memcpy(seg_v_scale + k * row, vs.data() + so, row * 4);
    } else if (seg_k_scale || seg_v_scale) {
      // single-entry segment: its scale row is |x|/127 of its member's row
      int member = -1;
      for (int i = 0; i < n && member < 0; ++i)
        if (sg[i] == id) member = i;
      const size_t src = (size_t)slot[member] * row;
      for (size_t r = 0; r < row; ++r) {
        if (seg_k_scale) single(__half2float(kf[src + r]), seg_k_scale + k * row + r);
        if (seg_v_scale) single(__half2float(vf[src + r]), seg_v_scale + k * row + r);
      }
    }
    if (seg_count) seg_count[k] = sc[id];
  }
  (void)n8;
  return CKV_OK;
}

int ckv_read_staged(ckv_engine* eng, int32_t layer, int32_t seq, int32_t count, double* mass, void* stream) {
  if (!eng || !mass) return fail(CKV_EINVAL, "null argument");
  const ckv::Dev& d = eng->d;
  if (layer < 0 || layer >= d.L || seq < 0 || seq >= d.B) return fail(CKV_EINVAL, "bad (layer, seq)");
  if (count < 0 || count > d.cap) return fail(CKV_EINVAL, "count %d outside [0, capacity]", count);
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "ckv_read_staged sync");
  const int c = layer * d.B + seq;
  if (count > 0) e = cudaMemcpy(mass, d.abar + (size_t)c * d.cap, (size_t)count * 8, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? CKV_OK : cuda_fail(e, "ckv_read_staged copy");
}

}  // extern "C"
