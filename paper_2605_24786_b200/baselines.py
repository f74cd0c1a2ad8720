"""Comparison policies on the B200 engine — the drop-in for the
reference's `baselines.py` (full cache, sliding window, heavy hitter, matched-rate
replay), running on the same device caches and the same K2/K3 kernels as Conf-KV:
K3's victim keys switch by policy (cumulative attention for the heavy hitter, the
storage index for the sliding window, alpha = 0 / 1 composites or host-drawn victims for
the matched-rate modes), everything else — the order-preserving compaction, the kept
maps, the records — is shared. The comparison policies never quantize (they only call
DecodePolicy.__init__ in the reference).

Batched like ConfKVEngine: every sequence runs the same policy; a matched-rate replay
applies its schedule to every sequence, and its random mode draws each sequence's
victims from its own `SeededRng(config.seed).spawn("vict")` stream (one reference
policy instance per sequence).
"""

from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from .config import ModelShape, PolicyConfig
from .engine import ConfKVEngine, EvictionEvent

CUM_ATTENTION = "cum_attention"
MATCHED_MODES = ("random", "recency_only", "attention_only")

_U64 = (1 << 64) - 1
_GAMMA, _M1, _M2 = 0x9E3779B97F4B7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB


def _mix(x: int) -> int:
    x = ((x ^ (x >> 30)) * _M1) & _U64
    x = ((x ^ (x >> 27)) * _M2) & _U64
    return x ^ (x >> 31)


def mix_u64(*parts: int) -> int:
    """rng.py:34-40."""
    acc = 0
    for p in parts:
        acc = _mix((acc + (p & _U64) + _GAMMA) & _U64)
    return acc


class SeededRng:
    """The counter-based SplitMix64 stream of rng.py:43-105 (draws the matched-rate
    random victims on the host, exactly as the reference does)."""

    def __init__(self, seed: int):
        self.seed = int(seed) & _U64
        self.counter = 0

    def next_u64(self) -> int:
        self.counter += 1
        return _mix((self.seed + self.counter * _GAMMA) & _U64)

    def integers(self, high: int) -> int:
        if high <= 0:
            raise ValueError(f"high must be positive, got {high}")
        return (self.next_u64() * high) >> 64

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


class FullCachePolicy(ConfKVEngine):
    """No eviction; the reference memory ceiling (baselines.py:68-77)."""

    name = "full"
    _policy = _lib.POLICY_FULL

    def __init__(self, config: PolicyConfig, shape: ModelShape, *, batch: int = 1, capacity: int,
                 device=None):
        super().__init__(config, shape, quantize=False, batch=batch, capacity=capacity, device=device)
        self.name = "full"

    def _record_budget(self, sq):
        return None


class SlidingWindowPolicy(ConfKVEngine):
    """Fixed recency window (baselines.py:80-94, sliding_window_step :21-31)."""

    _policy = _lib.POLICY_SLIDING

    def __init__(self, config: PolicyConfig, shape: ModelShape, window: int = 512, *, batch: int = 1,
                 capacity: int | None = None, device=None):
        if window < 1:
            raise ValueError(f"window must be >= 1, got {window}")
        self.window = int(window)
        self._policy_param = self.window
        cap = capacity if capacity is not None else max(self.window, config.n_low) + 2
        super().__init__(config, shape, quantize=False, batch=batch, capacity=cap, device=device)
        self.name = f"sliding-{window}"

    def _record_budget(self, sq):
        return self.window


class HeavyHitterPolicy(ConfKVEngine):
    """Cumulative attention + protected recent window (baselines.py:97-113,
    heavy_hitter_step :34-54, accumulate_attention :57-65). The device `ema` column holds
    the aux channel CUM_ATTENTION (`read_cache(...)["cum"]`)."""

    _policy = _lib.POLICY_HEAVY_HITTER

    def __init__(self, config: PolicyConfig, shape: ModelShape, cap: int | None = None, *, batch: int = 1,
                 capacity: int | None = None, device=None):
        self.cap = int(cap) if cap is not None else config.n_low
        if self.cap < config.protected_p:
            raise ValueError(f"cap {self.cap} smaller than protected window {config.protected_p}")
        self._policy_param = self.cap
        c = capacity if capacity is not None else max(self.cap, config.n_low) + 2
        super().__init__(config, shape, quantize=False, batch=batch, capacity=c, device=device)
        self.name = f"heavy-hitter-{self.cap}"

    def _record_budget(self, sq):
        return self.cap

    def read_cache(self, layer: int, seq: int = 0, stream=None) -> dict:
        r = super().read_cache(layer, seq, stream)
        r["cum"] = r["ema"]
        r["ema"] = np.zeros_like(r["ema"])   # the reference never updates the EMA here
        return r


def write_schedule(events, path) -> None:
    """baselines.py:119-125 — JSONL of {step, layer, evict_count}."""
    with open(path, "w") as f:
        for e in events:
            f.write(json.dumps({"step": e.step, "layer": e.layer, "evict_count": e.evict_count}) + "\n")


def read_schedule(path) -> list[EvictionEvent]:
    """baselines.py:128-136."""
    out = []
    with open(path) as f:
        for line in f:
            if line.strip():
                d = json.loads(line)
                out.append(EvictionEvent(d["step"], d["layer"], d["evict_count"]))
    return out


class MatchedRatePolicy(ConfKVEngine):
    """Replay a recorded eviction schedule, changing only how victims are picked
    (baselines.py:141-191): uniformly at random (host SeededRng, uploaded with
    ckv_set_victims), by recency alone (alpha = 0) or by attention alone (alpha = 1)."""

    def __init__(self, config: PolicyConfig, shape: ModelShape, schedule, mode: str, *, batch: int = 1,
                 capacity: int | None = None, device=None):
        if mode not in MATCHED_MODES:
            raise ValueError(f"mode must be one of {MATCHED_MODES}, got {mode!r}")
        self.mode = mode
        self._policy = {"random": _lib.POLICY_MATCHED_RANDOM, "recency_only": _lib.POLICY_MATCHED_RECENCY,
                        "attention_only": _lib.POLICY_MATCHED_ATTENTION}[mode]
        self._events: dict[tuple[int, int], int] = {}
        for e in schedule:
            st, layer, cnt = (e.step, e.layer, e.evict_count) if isinstance(e, EvictionEvent) else e
            if (st, layer) in self._events:
                raise ValueError(f"duplicate schedule event for step {st} layer {layer}")
            self._events[(st, layer)] = int(cnt)
        super().__init__(config, shape, quantize=False, batch=batch, capacity=capacity, device=device)
        self.name = f"matched-{mode.replace('_', '-')}"
        L, B = shape.num_layers, self.batch
        self._hlen = np.zeros((L, B), np.int64)    # host mirror of valid_len (deterministic here)
        self._rngs = [SeededRng(config.seed).spawn(0x76696374) for _ in range(B)]   # "vict"
        self._counts = (C.c_int32 * (L * B))()

    def _record_budget(self, sq):
        return None

    def prefill(self, k, v, first_pos: int = 0, layer_begin: int = 0, stream=None) -> None:
        super().prefill(k, v, first_pos, layer_begin, stream)
        self._hlen[layer_begin:layer_begin + k.shape[0]] += k.shape[2]

    def _pre_manage(self, step: int, stream) -> None:
        L, B, P = self.shape.num_layers, self.batch, self.config.protected_p
        counts = np.zeros((L, B), np.int32)
        for layer in range(L):
            counts[layer, :] = self._events.get((step, layer), 0)
        vic = None
        if self.mode == "random":
            maxv = max(1, int(counts.max()))
            vic = np.zeros((L, B, maxv), np.int32)
            for b in range(B):                       # each sequence's own stream, layer order
                for layer in range(L):
                    cnt = int(counts[layer, b])
                    if cnt:
                        ncand = int(self._hlen[layer, b]) - P
                        if cnt > ncand:
                            raise ValueError(f"schedule demands {cnt} evictions but only {ncand} candidates")
                        vic[layer, b, :cnt] = self._rngs[b].choice_without_replacement(ncand, cnt)
        self._counts_keep = counts
        self._vic_keep = vic
        s = C.c_void_p((stream if stream is not None else __import__("torch").cuda.current_stream()).cuda_stream)
        _lib.check(self.lib.ckv_set_victims(self._h, C.c_void_p(counts.ctypes.data),
                                            None if vic is None else C.c_void_p(vic.ctypes.data),
                                            0 if vic is None else vic.shape[2], s))
        # valid_len after this step: count evicted, one appended
        self._hlen += 1 - np.minimum(counts, np.maximum(self._hlen - P, 0))


__all__ = ["FullCachePolicy", "SlidingWindowPolicy", "HeavyHitterPolicy", "MatchedRatePolicy", "EvictionEvent",
           "write_schedule", "read_schedule", "SeededRng", "CUM_ATTENTION", "MATCHED_MODES"]
