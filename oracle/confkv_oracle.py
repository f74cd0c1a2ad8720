"""CPU ORACLE for the Conf-KV per-step cache-manager hot path.

TEST INFRASTRUCTURE ONLY. This module restates, in NumPy, the arithmetic of
the reference (`/root/reference/pkg/src/confkv`, a pure-Python/NumPy package)
so that the GPU path can be checked on the GPU box, where the reference does
not exist. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU arms
may import it, and only as the checker / the timed CPU baseline. The product
path (`paper_2605_24786_b200`) never imports it and has no CPU fallback.

Pinning: `tests/golden/make_golden.py` imports the real reference in the build
container, runs it on seeded inputs and stores inputs + outputs as fixtures;
`tests/test_oracle_golden.py` checks this restatement against every fixture
(bit-exact for EMA, kept sets, codes, scales, records; the reference's own
arithmetic is reproduced op for op, so equality is exact, not approximate).

Generalisation: the reference is MHA-only. This oracle stores K/V per KV head
(GQA); query head j reads KV head j // group. With group == 1 it is the
reference; with group > 1 it equals the reference run on K/V repeated across
each group (checked by the golden fixtures), except that `memory_bytes`
counts KV heads, not the expanded query heads.

Each function cites the reference lines it follows.
"""

from __future__ import annotations

import math

import numpy as np

HIGH = -1          # cache.py:20 precision tag of unquantized entries
P2_FLOOR = 1e-12   # confidence.py:19


# ----------------------------------------------------------------------------
# confidence (K1)
# ----------------------------------------------------------------------------

def softmax64(logits, temperature=None) -> np.ndarray:
    """policy.py:175-179 (optional /T) then confidence.py:31-39."""
    x = np.asarray(logits, dtype=np.float64)
    if temperature is not None:
        x = x / temperature
    if x.ndim != 1 or x.shape[0] < 2:
        raise ValueError(f"need a vector of at least 2 logits, got shape {x.shape}")
    if not np.all(np.isfinite(x)):
        raise ValueError("logits must all be finite")
    e = np.exp(x - x.max())
    return e / e.sum()


def confidence(p: np.ndarray, weights=(0.4, 0.3, 0.3)) -> dict:
    """confidence.py:42-82 — entropy/ln V, top-2 margin with the 1e-12 floor,
    sigmoid, top probability, weighted composite."""
    p = np.asarray(p, dtype=np.float64)
    if p.ndim != 1 or p.shape[0] < 2:
        raise ValueError("need a distribution over at least 2 tokens")
    if abs(p.sum() - 1.0) > 1e-6:
        raise ValueError("probabilities must sum to 1 within 1e-6")
    if np.any(p < 0):
        raise ValueError("probabilities must be nonnegative")
    pos = p[p > 0]
    h = float(-(pos * np.log(pos)).sum())
    h_norm = h / np.log(p.shape[0])
    two = np.partition(p, -2)[-2:]
    p1 = float(two[1])
    p2 = max(float(two[0]), P2_FLOOR)
    margin = max(np.log(p1) - np.log(p2), 0.0)
    sig = float(1.0 / (1.0 + np.exp(-margin)))
    wh, wm, wp = weights
    score = wh * (1.0 - h_norm) + wm * sig + wp * p1
    return {"entropy_norm": float(h_norm), "margin": float(margin), "margin_sig": sig,
            "top_prob": p1, "score": float(score)}


def select_tier(score: float, n_high: int, n_low: int, tau: float) -> int:
    """confidence.py:85-87 — c == tau is confident."""
    return n_high if score >= tau else n_low


def pyramid_budget(layer: int, num_layers: int, n0: int, beta: float, n_min: int) -> int:
    """policy.py:130-137."""
    return max(n_min, math.floor(n0 * beta ** (layer / num_layers)))


# ----------------------------------------------------------------------------
# INT8 quantizer (part of K4)
# ----------------------------------------------------------------------------

def quantize_lanes(x: np.ndarray):
    """quantizer.py:16-34. x [m, H, D] float32 -> (codes int8, scale f32 [H, D]).
    scale = amax/127 (f32), s = x/safe, code = copysign(floor(|s|+0.5), s),
    clipped to +-127; all-zero lanes get code 0."""
    x = np.asarray(x, dtype=np.float32)
    if x.ndim != 3 or x.shape[0] < 1:
        raise ValueError("expected [n_tokens, heads, head_dim] with n >= 1")
    if not np.all(np.isfinite(x)):
        raise ValueError("values must be finite")
    scale = np.abs(x).max(axis=0) / 127.0
    s = x / np.where(scale > 0, scale, 1.0)
    codes = np.clip(np.copysign(np.floor(np.abs(s) + 0.5), s), -127, 127).astype(np.int8)
    codes[:, scale == 0] = 0
    return codes, scale.astype(np.float32)


# ----------------------------------------------------------------------------
# per-layer storage (cache.py) — grouped K/V heads
# ----------------------------------------------------------------------------

class OracleCache:
    """Restates `LayerCache` (cache.py:49-274) with `kv_heads` storage heads.

    Storage prefix [0, n) sorted by original position; token-major arrays.
    Segments are kept as a Python list and renumbered when they empty,
    exactly as `_drop_empty_segments` (cache.py:222-234) does.
    """

    def __init__(self, kv_heads: int, head_dim: int, capacity: int = 64):
        self.kv_heads, self.head_dim = kv_heads, head_dim
        self.n = 0
        self._alloc(capacity)
        self.seg_k: list[np.ndarray] = []   # per segment: K scale [Hkv, D] f32
        self.seg_v: list[np.ndarray] = []
        self.seg_count: list[int] = []

    def _alloc(self, cap):
        shp = (cap, self.kv_heads, self.head_dim)
        self.k = np.zeros(shp, np.float32)
        self.v = np.zeros(shp, np.float32)
        self.kc = np.zeros(shp, np.int8)
        self.vc = np.zeros(shp, np.int8)
        self.pos = np.zeros(cap, np.int64)
        self.step = np.zeros(cap, np.int64)
        self.ema = np.zeros(cap, np.float64)
        self.seen = np.zeros(cap, bool)
        self.seg = np.full(cap, HIGH, np.int32)
        self.cum = np.zeros(cap, np.float64)   # aux channel CUM_ATTENTION (baselines.py:16, cache.py:144-147)

    @property
    def capacity(self):
        return self.pos.shape[0]

    def _grow(self):
        """cache.py:83-109 — doubling; contents preserved."""
        old = (self.k, self.v, self.kc, self.vc, self.pos, self.step, self.ema, self.seen, self.seg, self.cum)
        self._alloc(self.capacity * 2)
        for dst, src in zip((self.k, self.v, self.kc, self.vc, self.pos, self.step,
                             self.ema, self.seen, self.seg, self.cum), old):
            dst[: src.shape[0]] = src

    def append(self, k, v, position: int, gen_step: int):
        """cache.py:111-132."""
        k = np.asarray(k, np.float32)
        v = np.asarray(v, np.float32)
        if k.shape != (self.kv_heads, self.head_dim) or v.shape != k.shape:
            raise ValueError("bad K/V shape")
        if self.n == self.capacity:
            self._grow()
        i = self.n
        self.k[i], self.v[i] = k, v
        self.pos[i], self.step[i] = position, gen_step
        self.ema[i], self.seen[i], self.seg[i], self.cum[i] = 0.0, False, HIGH, 0.0
        self.n = i + 1

    def bulk_append(self, k, v, pos0: int, step0: int):
        """n consecutive appends (cache.py:111-132) in one copy: positions
        pos0.., steps step0..; used to stage large prefills quickly."""
        k = np.asarray(k, np.float32)
        v = np.asarray(v, np.float32)
        m = k.shape[0]
        while self.n + m > self.capacity:
            self._grow()
        sl = slice(self.n, self.n + m)
        self.k[sl], self.v[sl] = k, v
        self.pos[sl] = np.arange(pos0, pos0 + m)
        self.step[sl] = np.arange(step0, step0 + m)
        self.ema[sl], self.seen[sl], self.seg[sl], self.cum[sl] = 0.0, False, HIGH, 0.0
        self.n += m

    def dequant_kv(self, lo: int, hi: int):
        """cache.py:238-252 + quantizer.py:37-39: INT8 rows = code(f32) * scale(f32)."""
        k = self.k[lo:hi].copy()
        v = self.v[lo:hi].copy()
        tags = self.seg[lo:hi]
        for t in np.unique(tags[tags != HIGH]):
            rows = tags == t
            k[rows] = self.kc[lo:hi][rows].astype(np.float32) * self.seg_k[t]
            v[rows] = self.vc[lo:hi][rows].astype(np.float32) * self.seg_v[t]
        return k, v

    def ema_update(self, rows: np.ndarray, lam: float):
        """cache.py:151-177 — head mean (sequential fp64 sum / H), cold start,
        lam*ema + (1-lam)*mean; every live entry becomes seen."""
        a = np.asarray(rows, np.float64)
        if a.shape[1] != self.n:
            raise ValueError("attention rows do not match valid_len")
        if np.any(np.abs(a.sum(axis=1) - 1.0) > 1e-4):
            raise ValueError("attention rows must each sum to 1 within 1e-4")
        mean = a.mean(axis=0)
        n = self.n
        seen = self.seen[:n]
        ema = self.ema[:n]
        ema[~seen] = mean[~seen]
        ema[seen] = lam * ema[seen] + (1.0 - lam) * mean[seen]
        self.seen[:n] = True

    def compact(self, keep: np.ndarray) -> int:
        """cache.py:181-234 — order-preserving gather, member accounting,
        empty-segment drop with renumbering."""
        keep = np.asarray(keep, bool)
        gone = int((~keep).sum())
        if gone == 0:
            return 0
        n = self.n
        for tag in self.seg[:n][~keep]:
            if tag != HIGH:
                self.seg_count[tag] -= 1
        idx = np.nonzero(keep)[0]
        m = idx.shape[0]
        for arr in (self.k, self.v, self.kc, self.vc, self.pos, self.step, self.ema, self.seen, self.seg,
                    self.cum):
            arr[:m] = arr[idx]
        self.n = m
        if self.seg_count and any(c == 0 for c in self.seg_count):
            remap = np.full(len(self.seg_count), HIGH, np.int32)
            live = [i for i, c in enumerate(self.seg_count) if c > 0]
            remap[live] = np.arange(len(live), dtype=np.int32)
            tags = self.seg[:m]
            q = tags != HIGH
            tags[q] = remap[tags[q]]
            self.seg_k = [self.seg_k[i] for i in live]
            self.seg_v = [self.seg_v[i] for i in live]
            self.seg_count = [self.seg_count[i] for i in live]
        return gone

    def quantize_window(self, window: int, t: int) -> int:
        """quantizer.py:42-68 — HIGH entries with step <= t - W join ONE new segment."""
        n = self.n
        if n == 0:
            return 0
        aged = (self.seg[:n] == HIGH) & (self.step[:n] <= t - window)
        cnt = int(aged.sum())
        if cnt == 0:
            return 0
        rows = np.nonzero(aged)[0]
        kc, ks = quantize_lanes(self.k[rows])
        vc, vs = quantize_lanes(self.v[rows])
        sid = len(self.seg_count)
        self.seg_k.append(ks)
        self.seg_v.append(vs)
        self.seg_count.append(cnt)
        self.kc[rows], self.vc[rows] = kc, vc
        self.seg[rows] = sid
        return cnt

    def int8_count(self) -> int:
        return int((self.seg[: self.n] != HIGH).sum())

    def memory_bytes(self) -> int:
        """cache.py:266-274 with KV heads as the storage heads."""
        elems = self.kv_heads * self.head_dim
        n8 = self.int8_count()
        return ((self.n - n8) * 2 + n8) * elems * 2 + len(self.seg_count) * 4 * elems * 2


# ----------------------------------------------------------------------------
# attention (K2)
# ----------------------------------------------------------------------------

def attend(q: np.ndarray, cache: OracleCache, block: int = 128):
    """attention.py:60-102 — fp64 online softmax over blocks of `block`
    storage rows, INT8 rows dequantized on read. q [Hq, D] -> out [Hq, D],
    weights [Hq, n] (normalised), both fp64. GQA by repeating KV heads."""
    n = cache.n
    if n == 0:
        raise ValueError("attention over an empty cache")
    q = np.asarray(q, np.float64)
    hq, d = q.shape
    grp = hq // cache.kv_heads
    m = np.full(hq, -np.inf)
    z = np.zeros(hq)
    acc = np.zeros((hq, d))
    w = np.zeros((hq, n))
    inv = 1.0 / np.sqrt(d)
    for lo in range(0, n, block):
        hi = min(lo + block, n)
        kb, vb = cache.dequant_kv(lo, hi)
        if grp > 1:
            kb = np.repeat(kb, grp, axis=1)
            vb = np.repeat(vb, grp, axis=1)
        s = np.einsum("hd,nhd->hn", q, kb.astype(np.float64)) * inv
        m2 = np.maximum(m, s.max(axis=1))
        corr = np.exp(m - m2)
        e = np.exp(s - m2[:, None])
        z = z * corr + e.sum(axis=1)
        acc = acc * corr[:, None] + np.einsum("hn,nhd->hd", e, vb.astype(np.float64))
        w[:, :lo] *= corr[:, None]
        w[:, lo:hi] = e
        m = m2
    return acc / z[:, None], w / z[:, None]


# ----------------------------------------------------------------------------
# ranking / eviction (K3)
# ----------------------------------------------------------------------------

def _minmax(x: np.ndarray) -> np.ndarray:
    """policy.py:72-77."""
    lo, hi = x.min(), x.max()
    if hi == lo:
        return np.zeros_like(x, dtype=np.float64)
    return (x - lo) / (hi - lo)


def composite(ema: np.ndarray, steps: np.ndarray, alpha: float) -> np.ndarray:
    """policy.py:93-97 over the candidate prefix already sliced by the caller."""
    return alpha * _minmax(ema) + (1.0 - alpha) * _minmax(steps.astype(np.float64))


def victims(cache: OracleCache, count: int, protected: int, alpha: float) -> np.ndarray:
    """policy.py:80-114 — lowest (composite, index) among the first n - P slots."""
    n = cache.n
    if n <= protected:
        raise ValueError(f"no candidates: valid_len {n} <= protected_p {protected}")
    cut = n - protected
    comp = composite(cache.ema[:cut], cache.step[:cut], alpha)
    idx = np.arange(cut)
    return idx[np.lexsort((idx, comp))[:count]]


def evict(cache: OracleCache, budget: int, protected: int, alpha: float):
    """policy.py:117-127. Returns (evicted count, kept old indices)."""
    if budget < protected:
        raise ValueError(f"budget {budget} smaller than protected window {protected}")
    n = cache.n
    excess = n - budget
    if excess <= 0:
        return 0, np.arange(n)
    keep = np.ones(n, bool)
    keep[victims(cache, excess, protected, alpha)] = False
    kept = np.nonzero(keep)[0]
    return cache.compact(keep), kept


# ----------------------------------------------------------------------------
# the per-sequence engine (DecodePolicy + ConfKVEngine)
# ----------------------------------------------------------------------------

class OracleEngine:
    """policy.py:147-274 for one sequence.

    `cfg` is any object with the PolicyConfig field names (this repo's or the
    reference's). `kv_heads` defaults to `num_heads` (MHA).
    """

    def __init__(self, cfg, num_layers, num_heads, head_dim, vocab_size,
                 quantize=False, kv_heads=None, capacity=64):
        self.cfg = cfg
        self.L, self.H, self.D, self.V = num_layers, num_heads, head_dim, vocab_size
        self.Hkv = kv_heads or num_heads
        self.quantize = quantize
        self.caches = [OracleCache(self.Hkv, head_dim, capacity) for _ in range(num_layers)]
        self.prefill_len = 0

    def layer_budget(self, layer: int, tier: int) -> int:
        """policy.py:249-254."""
        c = self.cfg
        if not c.pyramid_enabled:
            return tier
        return pyramid_budget(layer, self.L, tier, c.pyramid_beta, c.pyramid_n_min)

    def begin_prefill(self, n: int):
        self.prefill_len = n

    def append_prefill(self, layer, k, v, position):
        """policy.py:165-168 — step = position - prefill_len (nonpositive)."""
        self.caches[layer].append(k, v, position, position - self.prefill_len)

    def attend(self, layer: int, q):
        return attend(q, self.caches[layer], self.cfg.block_size_b)

    def step(self, logits, rows, new_kv, t: int, return_kept=False):
        """policy.py:187-224 + 256-274, one sequence. Returns the StepRecord
        dict (policy.py:54-69), and the per-layer kept old-index arrays."""
        c = self.cfg
        if len(rows) != self.L or len(new_kv) != self.L:
            raise ValueError("attention_rows and new_kv must have one entry per layer")
        temp = c.temperature if c.sampling_mode == "temperature" else None
        p = softmax64(logits, temp)
        f = confidence(p, (c.w_entropy, c.w_margin, c.w_top))
        len_pre = [x.n for x in self.caches]
        tier = select_tier(f["score"], c.n_high, c.n_low, c.tau)
        len_post, evicted, int8, kept_all = [], [], [], []
        for layer, cache in enumerate(self.caches):
            cache.ema_update(rows[layer], c.ema_lambda)
            nl = self.layer_budget(layer, tier)
            prot = min(c.protected_p, nl)
            gone, kept = 0, np.arange(cache.n)
            if cache.n > nl:
                gone, kept = evict(cache, nl, prot, c.alpha)
            if self.quantize:
                cache.quantize_window(c.fp16_window_w, t)
            len_post.append(cache.n)
            evicted.append(gone)
            int8.append(cache.int8_count())
            kept_all.append(kept)
        position = self.prefill_len + t - 1
        for layer, cache in enumerate(self.caches):
            k, v = new_kv[layer]
            cache.append(k, v, position, t)
        token = int(np.argmax(p)) if c.sampling_mode == "greedy" else -1
        rec = {"step": t, "confidence": f["score"], "entropy_norm": f["entropy_norm"],
               "margin": f["margin"], "margin_sig": f["margin_sig"], "top_prob": f["top_prob"],
               "budget": tier, "len_pre": len_pre, "len_post": len_post, "evicted": evicted,
               "int8": int8, "memory_bytes": sum(x.memory_bytes() for x in self.caches),
               "token": token}
        return (rec, kept_all) if return_kept else rec


# ----------------------------------------------------------------------------
# comparison policies (baselines.py) over the same cache substrate
# ----------------------------------------------------------------------------

def sliding_window_step(cache: OracleCache, window_n: int) -> tuple[int, np.ndarray]:
    """baselines.py:21-31 — keep the window_n largest positions (a storage suffix)."""
    if window_n < 1:
        raise ValueError(f"window must be >= 1, got {window_n}")
    n = cache.n
    excess = n - window_n
    if excess <= 0:
        return 0, np.arange(n)
    keep = np.zeros(n, bool)
    keep[excess:] = True
    return cache.compact(keep), np.nonzero(keep)[0]


def accumulate_attention(cache: OracleCache, rows) -> None:
    """baselines.py:57-65 — cum[:n] += head mean."""
    a = np.asarray(rows, np.float64)
    if a.shape[1] != cache.n:
        raise ValueError("attention rows do not match valid_len")
    cache.cum[: cache.n] += a.mean(axis=0)


def heavy_hitter_step(cache: OracleCache, cap_n: int, protected_p: int) -> tuple[int, np.ndarray]:
    """baselines.py:34-54 — victims = lowest (cum, index) among the first n - P slots."""
    if cap_n < protected_p:
        raise ValueError(f"cap {cap_n} smaller than protected window {protected_p}")
    n = cache.n
    excess = n - cap_n
    if excess <= 0:
        return 0, np.arange(n)
    cut = n - protected_p
    cand = np.arange(cut)
    order = np.lexsort((cand, cache.cum[:cut]))
    keep = np.ones(n, bool)
    keep[cand[order[:excess]]] = False
    return cache.compact(keep), np.nonzero(keep)[0]


class SeededRng:
    """rng.py:43-105 (the parts the matched-rate baseline draws from)."""

    def __init__(self, seed: int):
        self.seed = int(seed) & ((1 << 64) - 1)
        self.counter = 0

    def _raw(self, n):
        ks = np.arange(self.counter + 1, self.counter + n + 1, dtype=np.uint64)
        self.counter += n
        with np.errstate(over="ignore"):
            return _mix(np.uint64(self.seed) + ks * _G)

    def integers(self, high: int) -> int:
        """rng.py:78-86 — multiply-shift (u64 * high) >> 64, one draw."""
        if high <= 0:
            raise ValueError(f"high must be positive, got {high}")
        return int((int(self._raw(1)[0]) * high) >> 64)

    def choice_without_replacement(self, population: int, k: int) -> np.ndarray:
        """rng.py:88-97 — partial Fisher-Yates."""
        if k > population:
            raise ValueError(f"cannot draw {k} from {population}")
        idx = np.arange(population, dtype=np.int64)
        for i in range(k):
            j = i + self.integers(population - i)
            idx[i], idx[j] = idx[j], idx[i]
        return idx[:k]

    def spawn(self, tag: int) -> "SeededRng":
        return SeededRng(mix_u64(self.seed, tag))


MATCHED_MODES = ("random", "recency_only", "attention_only")


class OracleBaseline(OracleEngine):
    """baselines.py:68-191 for one sequence: kind in {"full", "sliding", "heavy_hitter",
    "matched"}; never quantizes (the baselines call DecodePolicy.__init__ only)."""

    def __init__(self, cfg, num_layers, num_heads, head_dim, vocab_size, kind, *, window=512, cap=None,
                 schedule=None, mode=None, kv_heads=None, capacity=64):
        super().__init__(cfg, num_layers, num_heads, head_dim, vocab_size, quantize=False,
                         kv_heads=kv_heads, capacity=capacity)
        self.kind = kind
        self.window = window
        self.cap = cap if cap is not None else cfg.n_low
        if kind == "matched":
            if mode not in MATCHED_MODES:
                raise ValueError(f"mode must be one of {MATCHED_MODES}, got {mode!r}")
            self.mode = mode
            self.events = {}
            for st, layer, cnt in schedule:
                if (st, layer) in self.events:
                    raise ValueError(f"duplicate schedule event for step {st} layer {layer}")
                self.events[(st, layer)] = cnt
            self.victim_rng = SeededRng(cfg.seed).spawn(0x76696374)   # "vict"

    def _manage(self, rows, t):
        """The subclass _manage bodies (baselines.py:73-191). Returns (budget, kept per layer)."""
        c = self.cfg
        kept_all, budget = [], None
        for layer, cache in enumerate(self.caches):
            gone, kept = 0, np.arange(cache.n)
            if self.kind == "sliding":
                gone, kept = sliding_window_step(cache, self.window)
                budget = self.window
            elif self.kind == "heavy_hitter":
                accumulate_attention(cache, rows[layer])
                gone, kept = heavy_hitter_step(cache, self.cap, c.protected_p)
                budget = self.cap
            elif self.kind == "matched":
                cache.ema_update(rows[layer], c.ema_lambda)
                count = self.events.get((t, layer), 0)
                if count:
                    ncand = cache.n - c.protected_p
                    if count > ncand:
                        raise ValueError(f"schedule demands {count} evictions but only {ncand} candidates")
                    if self.mode == "random":
                        vic = self.victim_rng.choice_without_replacement(ncand, count)
                    else:
                        vic = victims(cache, count, c.protected_p, 0.0 if self.mode == "recency_only" else 1.0)
                    keep = np.ones(cache.n, bool)
                    keep[vic] = False
                    kept = np.nonzero(keep)[0]
                    gone = cache.compact(keep)
            kept_all.append((gone, kept))
        return budget, kept_all

    def step(self, logits, rows, new_kv, t: int, return_kept=False):
        c = self.cfg
        if len(rows) != self.L or len(new_kv) != self.L:
            raise ValueError("attention_rows and new_kv must have one entry per layer")
        temp = c.temperature if c.sampling_mode == "temperature" else None
        p = softmax64(logits, temp)
        f = confidence(p, (c.w_entropy, c.w_margin, c.w_top))
        len_pre = [x.n for x in self.caches]
        budget, ka = self._manage(rows, t)
        len_post = [x.n for x in self.caches]
        position = self.prefill_len + t - 1
        for layer, cache in enumerate(self.caches):
            k, v = new_kv[layer]
            cache.append(k, v, position, t)
        token = int(np.argmax(p)) if c.sampling_mode == "greedy" else -1
        rec = {"step": t, "confidence": f["score"], "entropy_norm": f["entropy_norm"],
               "margin": f["margin"], "margin_sig": f["margin_sig"], "top_prob": f["top_prob"],
               "budget": budget, "len_pre": len_pre, "len_post": len_post, "evicted": [g for g, _ in ka],
               "int8": [0] * self.L, "memory_bytes": sum(x.memory_bytes() for x in self.caches),
               "token": token}
        return (rec, [k for _, k in ka]) if return_kept else rec


# ----------------------------------------------------------------------------
# SplitMix64 (rng.py) — only for seeded synthetic inputs shared by both sides
# ----------------------------------------------------------------------------

_G = np.uint64(0x9E3779B97F4B7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(x):
    """rng.py:28-31."""
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def mix_u64(*parts: int) -> int:
    """rng.py:34-40."""
    acc = np.uint64(0)
    with np.errstate(over="ignore"):
        for p in parts:
            acc = _mix((acc + np.uint64(p & 0xFFFFFFFFFFFFFFFF)) * np.uint64(1) + _G)
    return int(acc)


def splitmix_normal(seed: int, n: int) -> np.ndarray:
    """rng.py:43-55 + 73-84: draws 1..2*ceil(n/2) of stream `seed` -> Box-Muller."""
    pairs = (n + 1) // 2
    ks = np.arange(1, 2 * pairs + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        raw = _mix(np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + ks * _G)
    u = (raw >> np.uint64(11)).astype(np.float64) * float(2.0 ** -53)
    u1 = np.maximum(u[:pairs], float(2.0 ** -53))
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * np.pi * u[pairs:]
    return np.concatenate([r * np.cos(th), r * np.sin(th)])[:n]


# ----------------------------------------------------------------------------
# vocab-sharded confidence: restatement of K1's online tuple + rank-order merge
# (checker for the sharded path; the unsharded reference is confidence() above)
# ----------------------------------------------------------------------------

def online_tuple(logits_slice, offset: int, temperature=None):
    """(m, Z, S, top1, top2, argmax) of one vocab slice, Z/S relative to m."""
    x = np.asarray(logits_slice, dtype=np.float64)
    if temperature is not None:
        x = x / temperature
    m = x.max()
    e = np.exp(x - m)
    two = np.partition(x, -2)[-2:] if x.shape[0] > 1 else np.array([-np.inf, x[0]])
    return (m, e.sum(), ((x - m) * e).sum(), two[1], two[0], offset + int(np.argmax(x)))


def merge_tuples(tuples, vocab_total: int, weights=(0.4, 0.3, 0.3)) -> dict:
    """Rank-order merge of online_tuple()s and the confidence features (confidence.py:64-75)."""
    M = max(t[0] for t in tuples)
    Z = sum(t[1] * np.exp(t[0] - M) for t in tuples)
    S = sum(np.exp(t[0] - M) * (t[2] + (t[0] - M) * t[1]) for t in tuples)
    vals = sorted([v for t in tuples for v in (t[3], t[4])], reverse=True)
    top = max(t[3] for t in tuples)
    arg = min(t[5] for t in tuples if t[3] == top)
    h_norm = (np.log(Z) - S / Z) / np.log(vocab_total)
    p1 = 1.0 / Z
    p2 = max(np.exp(vals[1] - M) / Z, P2_FLOOR)
    margin = max(np.log(p1) - np.log(p2), 0.0)
    sig = 1.0 / (1.0 + np.exp(-margin))
    wh, wm, wp = weights
    return {"entropy_norm": h_norm, "margin": margin, "margin_sig": sig, "top_prob": p1,
            "score": wh * (1.0 - h_norm) + wm * sig + wp * p1, "argmax": arg}


# ----------------------------------------------------------------------------
# decode driver model (F1 checker)
# ----------------------------------------------------------------------------

def reference_forward(token: int, kv: list, weights: dict, num_heads: int, head_dim: int, q_dtype=None):
    """ReferenceModel.forward (simulator.py:58-92) in fp64 over given cache contents.
    kv[layer] = (keys [n, Hkv, D], values [n, Hkv, D]) of the pre-step cache (n may be 0:
    the layer then contributes nothing, :84-90); weights as DecodeModel names them
    (w_q [L,d,Hq*D], w_k/w_v [L,d,Hkv*D], w_o [L,Hq*D,d], w_out [d,V], embedding [V,d]).
    GQA: K/V heads repeated over each query-head group. `q_dtype` rounds q to the
    engine's query input type (fp16) before the attention. Returns (logits [V],
    per-layer attention outputs [Hq, D], per-layer new (k, v) [Hkv, D])."""
    h, hd = num_heads, head_dim
    x = np.asarray(weights["embedding"][int(token)], np.float64).copy()
    outs, new_kv = [], []
    for layer, (keys, values) in enumerate(kv):
        q = (x @ np.asarray(weights["w_q"][layer], np.float64)).reshape(h, hd)
        if q_dtype is not None:
            q = q.astype(q_dtype).astype(np.float64)
        k = x @ np.asarray(weights["w_k"][layer], np.float64)
        v = x @ np.asarray(weights["w_v"][layer], np.float64)
        hkv = k.size // hd
        k, v = k.reshape(hkv, hd), v.reshape(hkv, hd)
        if len(keys):
            kb = np.repeat(np.asarray(keys, np.float64), h // hkv, axis=1)
            vb = np.repeat(np.asarray(values, np.float64), h // hkv, axis=1)
            s = np.einsum("hd,nhd->hn", q, kb) / np.sqrt(hd)
            e = np.exp(s - s.max(axis=1, keepdims=True))
            out = np.einsum("hn,nhd->hd", e / e.sum(axis=1, keepdims=True), vb)
            x = x + out.reshape(-1) @ np.asarray(weights["w_o"][layer], np.float64)
        else:
            out = np.zeros((h, hd))
        outs.append(out)
        new_kv.append((k, v))
    return x @ np.asarray(weights["w_out"], np.float64), outs, new_kv
