"""`ConfKVEngine` on B200 — the drop-in for the reference's per-step cache
manager (`confkv.policy.ConfKVEngine`, policy.py:230-274, with
`DecodePolicy.step`, policy.py:187-224) batched over `batch` sequences.

PyTorch is plumbing here (device tensors, the current stream); every byte of
the hot path is touched by the sm_100a kernels behind the C ABI
(`include/confkv_b200.h`). Call shapes, argument meaning and exceptions
follow the reference:

    eng = ConfKVEngine(cfg, ModelShape(...), quantize=True, batch=8)
    eng.begin_prefill(n); eng.prefill(k, v)            # DecodePolicy.begin/append_prefill
    out = eng.attend(layer, q)                         # tiled_attention per layer (pure)
    res = eng.step(logits, k_new, v_new, step=t)       # DecodePolicy.step
    # or fused: eng.step(logits, k_new, v_new, step=t, q=q_all_layers)
    recs = eng.records()                               # StepRecord per sequence (syncs)

Reference-signature path (attention rows supplied by the caller, as in the
reference's trace driver): `eng.step_rows(logits, attention_rows, new_kv, t)`.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import ConfigError, ModelShape, PolicyConfig, budget_table


@dataclass
class StepRecord:
    """One trace row for one sequence (policy.py:36-69)."""

    step: int
    confidence: float
    entropy_norm: float
    margin: float
    margin_sig: float
    top_prob: float
    budget: int | None
    len_pre: list[int]
    len_post: list[int]
    evicted: list[int]
    int8: list[int]
    memory_bytes: int
    token: int

    def to_dict(self) -> dict:
        return dict(self.__dict__)


@dataclass
class EvictionEvent:
    """One (step, layer, count) of a recorded eviction schedule (policy.py:140-144)."""

    step: int
    layer: int
    evict_count: int


@dataclass
class StepResult:
    out: torch.Tensor | None        # [L, B, Hq, D] fp32 attention outputs (when q was given)
    kept_map: torch.Tensor | None   # [L, B, capacity] int32: old storage index of survivor j
    kept_len: torch.Tensor | None   # [L, B] int32
    victims: torch.Tensor | None = None   # [L, B, capacity] int32: evicted old indices, ascending


class VictimList:
    """`kept=VictimList(buf)`: the kept-index map in compact form -- K3 writes each cache's
    evicted pre-step storage indices, ascending, to buf [L, B, capacity] int32 (the first
    `evicted` of the step's record are valid); the kept map is their complement in
    [0, len_pre) (policy.py:117-127). One int per cache in the steady state."""

    def __init__(self, buf: torch.Tensor):
        self.buf = buf


def kept_from_victims(len_pre: int, victims) -> np.ndarray:
    """The kept-index map of one cache from its victim list (ascending old indices)."""
    keep = np.ones(int(len_pre), bool)
    keep[np.asarray(victims, np.int64)] = False
    return np.nonzero(keep)[0].astype(np.int32)


class KeptMaps:
    """One step's kept-index maps on the host, held in their compact form: per (layer, seq)
    the pre-step length and the ascending victim list (policy.py:117-127, cache.py:206).
    `maps[layer][seq]` materialises that cache's kept map (the complement of its victims in
    [0, len_pre)) on access; `victims(layer, seq)` is the compact form itself."""

    def __init__(self, len_pre: np.ndarray, evicted: np.ndarray, head: np.ndarray, overflow: dict):
        # head [L, B, vmax]: the first victims of every cache; overflow[(l, b)]: the full list of
        # a cache that evicted more than vmax (a tier switch, step 1)
        self.len_pre, self.evicted, self._head, self._over = len_pre, evicted, head, overflow

    def victims(self, layer: int, seq: int) -> np.ndarray:
        v = self._over.get((layer, seq))
        return v if v is not None else self._head[layer, seq, :self.evicted[layer, seq]]

    def __len__(self) -> int:
        return self.len_pre.shape[0]

    def __getitem__(self, layer: int) -> list[np.ndarray]:
        return [kept_from_victims(self.len_pre[layer, b], self.victims(layer, b))
                for b in range(self.len_pre.shape[1])]

    def __iter__(self):
        return (self[layer] for layer in range(len(self)))


_DTYPES = {torch.float32: _lib.DTYPE_F32, torch.bfloat16: _lib.DTYPE_BF16, torch.float64: _lib.DTYPE_F64}


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _on(stream):
    """Run host-input conversions (H2D copies, casts) on the stream the kernels are launched
    on, so they are ordered before the launch whatever torch's current stream is."""
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


class LayerCacheView:
    """`policy.caches[layer]` of one sequence: the two fields the reference's drivers read
    (`valid_len`, `positions`; simulator.py:134-146, 433, 464-467). Host views of device
    state, read on access (synchronising) unless the engine's host mirror is fresh."""

    def __init__(self, engine: "ConfKVEngine", layer: int, seq: int = 0):
        self._e, self.layer, self.seq = engine, layer, seq

    @property
    def valid_len(self) -> int:
        return self._e._valid_len(self.layer, self.seq)

    @property
    def positions(self) -> np.ndarray:
        return self._e._positions(self.layer, self.seq)

    def __len__(self) -> int:
        return self.valid_len


class ConfKVEngine:
    """Batched Conf-KV cache manager on one GPU (policy.py:230-274)."""

    _policy = _lib.POLICY_CONFKV   # comparison policies (baselines.py) set their own
    _policy_param = 0

    def __init__(self, config: PolicyConfig, shape: ModelShape, quantize: bool = False,
                 record_schedule: bool = False, *, batch: int = 1, capacity: int | None = None,
                 max_segments: int | None = None, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("ConfKVEngine needs a CUDA device (B200); there is no CPU fallback")
        self.lib = _lib.load()
        self.config, self.shape, self.quantize = config, shape, bool(quantize)
        self.batch = int(batch)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        table = budget_table(config, shape)
        max_budget = max(max(r) for r in table)
        self.capacity = int(capacity) if capacity is not None else max_budget + 2
        self.name = "confkv-l" if config.pyramid_enabled else ("confkv-int8" if quantize else "confkv")
        # record_schedule (policy.py:238, 266-268): EvictionEvents per sequence, filled by
        # records() (call it every step); `schedule` is sequence 0's, the reference's view
        self.schedules = [[] for _ in range(self.batch)] if record_schedule else None
        self.schedule = self.schedules[0] if record_schedule else None
        self.budgets = table
        cfg = _lib.CkvConfig(
            tau=config.tau, n_high=config.n_high, n_low=config.n_low, protected_p=config.protected_p,
            fp16_window_w=config.fp16_window_w, block_size_b=config.block_size_b, alpha=config.alpha,
            ema_lambda=config.ema_lambda, w_entropy=config.w_entropy, w_margin=config.w_margin,
            w_top=config.w_top, quantize=int(self.quantize),
            temperature_mode=int(config.sampling_mode == "temperature"),
            temperature=float(config.temperature or 1.0),
            policy=int(self._policy), policy_param=int(self._policy_param))
        shp = _lib.CkvShape(shape.num_layers, shape.num_heads, shape.kv_heads, shape.head_dim, shape.vocab_size)
        tbl = (C.c_int32 * (2 * shape.num_layers))(*[x for row in table for x in row])
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.ckv_create(C.byref(cfg), C.byref(shp), self.batch, self.capacity,
                                           int(max_segments or 0), C.cast(tbl, C.c_void_p), C.byref(h)))
        self._h = h
        self.prefill_len = 0
        self.steps_run = 0
        L, B = shape.num_layers, self.batch
        self._kept_map = torch.empty((L, B, self.capacity), dtype=torch.int32, device=self.device)
        self._kept_len = torch.empty((L, B), dtype=torch.int32, device=self.device)
        self._rec_l = (_lib.CkvLayerRecord * (L * B))()
        self._rec_s = (_lib.CkvSeqRecord * B)()
        self._last_step = None
        self._next_t = 1          # mirror of the library's expected next step
        self._side = None
        # where K1 runs relative to K2 in step(q=...): "after" (default) / "before" = forked onto
        # a side stream, submitted after / before K2 (as ckv_step does); "serial" = after K2 on
        # the step's stream. Measured at Llama-8B 4K, batch 8: INT8 600 -> 575 us/step, FP16
        # 820 -> 797 us/step forked (tools/fork_probe.py).
        self._k1_order = os.environ.get("CKV_K1_ORDER", "after")
        self._rows_keep = [None] * L        # staged attention rows: one live tensor per layer
        self._host_len = np.zeros((L, B), np.int64)   # valid_len mirror (fresh after prefill / records())
        self._len_fresh = True
        self.caches_by_seq = [[LayerCacheView(self, layer, b) for layer in range(L)] for b in range(B)]

    @property
    def caches(self) -> list[LayerCacheView]:
        """The reference's `policy.caches` (policy.py:156-158): sequence 0's per-layer caches
        (the whole engine when batch == 1); `caches_by_seq[b]` for the others."""
        return self.caches_by_seq[0]

    def _valid_len(self, layer: int, seq: int) -> int:
        if not self._len_fresh:
            n = C.c_int32()
            nulls = [None] * 12
            _lib.check(self.lib.ckv_read_cache(self._h, layer, seq, C.byref(n), None, *nulls, _stream(None)))
            return int(n.value)
        return int(self._host_len[layer, seq])

    def _positions(self, layer: int, seq: int) -> np.ndarray:
        cap = self.capacity
        pos = np.zeros(cap, np.int64)
        n = C.c_int32()
        nulls = [None] * 11
        _lib.check(self.lib.ckv_read_cache(self._h, layer, seq, C.byref(n), None,
                                           pos.ctypes.data_as(C.c_void_p), *nulls, _stream(None)))
        return pos[: n.value]

    def read_staged(self, layer: int, seq: int, count: int, stream=None) -> np.ndarray:
        """Host copy of the head-mean attention mass staged for (layer, seq) by the last
        attend / stage (update_attention_ema's `mean`, cache.py:171), first `count` entries
        in pre-step storage order (synchronises). Parity hook."""
        out = np.zeros(max(int(count), 0), np.float64)
        _lib.check(self.lib.ckv_read_staged(self._h, layer, seq, int(count), out.ctypes.data_as(C.c_void_p),
                                            _stream(stream)))
        return out

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.ckv_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        return int(self.lib.ckv_device_bytes(self._h))

    @property
    def launch_count(self) -> int:
        """Kernels this engine has launched (graph-captured launches count once, at capture)."""
        return int(self.lib.ckv_launch_count(self._h))

    def reset(self, stream=None):
        _lib.check(self.lib.ckv_reset(self._h, _stream(stream)))
        self.steps_run = 0
        self._next_t = 1
        self._last_step = None
        self._host_len[:] = 0
        self._len_fresh = True

    # ------------------------------------------------------------------ inputs
    def _half(self, x, shape, name):
        if not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.asarray(x))
        x = x.to(device=self.device, dtype=torch.float16).contiguous()
        if tuple(x.shape) != tuple(shape):
            raise ValueError(f"expected {name} of shape {tuple(shape)}, got {tuple(x.shape)}")
        return x

    # ------------------------------------------------------------------ prefill
    def begin_prefill(self, prefill_len: int) -> None:
        """DecodePolicy.begin_prefill (policy.py:170-171)."""
        self.prefill_len = int(prefill_len)
        _lib.check(self.lib.ckv_begin_prefill(self._h, self.prefill_len))

    def prefill(self, k, v, first_pos: int = 0, layer_begin: int = 0, stream=None) -> None:
        """Bulk append_prefill: k, v [layers, batch, n, Hkv, D] (fp16) for positions
        first_pos..first_pos+n-1 of every sequence (policy.py:165-168)."""
        s = self.shape
        lc, n = k.shape[0], k.shape[2]
        with _on(stream):
            k = self._half(k, (lc, self.batch, n, s.kv_heads, s.head_dim), "prefill K")
            v = self._half(v, (lc, self.batch, n, s.kv_heads, s.head_dim), "prefill V")
        _lib.check(self.lib.ckv_prefill(self._h, layer_begin, lc, _ptr(k), _ptr(v), n, first_pos, _stream(stream)))
        if self.steps_run == 0 and self._len_fresh:
            self._host_len[layer_begin:layer_begin + lc] += n
        else:
            self._len_fresh = False

    def append_prefill(self, layer: int, k, v, position: int, stream=None) -> None:
        """DecodePolicy.append_prefill (policy.py:165-168): one entry per sequence,
        k/v [batch, Hkv, D] (or [Hkv, D] when batch == 1)."""
        s = self.shape
        k = torch.as_tensor(np.asarray(k)) if not isinstance(k, torch.Tensor) else k
        v = torch.as_tensor(np.asarray(v)) if not isinstance(v, torch.Tensor) else v
        if k.dim() == 2:
            k, v = k[None], v[None]
        self.prefill(k[None, :, None], v[None, :, None], first_pos=position, layer_begin=layer, stream=stream)

    # ------------------------------------------------------------------ attention
    def attend(self, layer: int, q, stream=None, weights: bool = False):
        """tiled_attention for one layer over every sequence (attention.py:60-102).
        q [batch, Hq, D] -> out [batch, Hq, D] fp32 (+ weights [batch, Hq, capacity])."""
        q = q if isinstance(q, torch.Tensor) else torch.as_tensor(np.asarray(q))
        if q.dim() == 2:
            q = q[None]
        out, w = self.attend_layers(q[None], layer, stream, weights)
        return (out[0], w[0]) if weights else out[0]

    def attend_layers(self, q, layer_begin: int = 0, stream=None, weights: bool = False, out=None, fork=None,
                      conf=None):
        # conf = (logits, dtype code, side stream): also this step's confidence pass (ckv_attend_conf)
        # fork (a torch stream): made to wait for the point where the attention grids are submitted,
        # before the combine (ckv_attend_fork), so work put on it next runs beside the combine
        s = self.shape
        lc = q.shape[0]
        with _on(stream):
            q = self._half(q, (lc, self.batch, s.num_heads, s.head_dim), "q")
        if out is None:
            out = torch.empty((lc, self.batch, s.num_heads, s.head_dim), dtype=torch.float32, device=self.device)
        elif (out.dtype != torch.float32 or tuple(out.shape) != (lc, self.batch, s.num_heads, s.head_dim)
              or not out.is_contiguous() or out.device != self.device):
            raise ValueError("out must be a contiguous fp32 device tensor [layers, batch, Hq, D]")
        if isinstance(weights, torch.Tensor):   # caller's buffer (fixed address: graph capture)
            if (weights.dtype != torch.float32 or tuple(weights.shape) != (lc, self.batch, s.num_heads, self.capacity)
                    or not weights.is_contiguous() or weights.device != self.device):
                raise ValueError("weights must be a contiguous fp32 device tensor [layers, batch, Hq, capacity]")
            w = weights
        else:
            w = (torch.zeros((lc, self.batch, s.num_heads, self.capacity), dtype=torch.float32, device=self.device)
                 if weights else None)
        if conf is not None:
            lg, dt, side = conf
            _lib.check(self.lib.ckv_attend_conf(self._h, layer_begin, lc, _ptr(q), _ptr(out), _ptr(w), _ptr(lg), dt,
                                                lg.stride(0), _stream(stream), C.c_void_p(side.cuda_stream)))
        elif fork is not None:
            _lib.check(self.lib.ckv_attend_fork(self._h, layer_begin, lc, _ptr(q), _ptr(out), _ptr(w), _stream(stream),
                                                C.c_void_p(fork.cuda_stream)))
        else:
            _lib.check(self.lib.ckv_attend(self._h, layer_begin, lc, _ptr(q), _ptr(out), _ptr(w), _stream(stream)))
        self._q_keep = q
        return out, w

    def stage_rows(self, layer: int, rows, stream=None) -> None:
        """Stage caller-supplied attention rows (the reference's `attention_rows[layer]`,
        [batch, Hq, n] fp64, or one [Hq, n_b] array per sequence) for the next step. Each
        sequence's rows must have exactly its valid_len entries and each row must sum to 1
        within 1e-4 (update_attention_ema, cache.py:164-170): a length mismatch is reported
        by the step's records (ValueError), a bad row sum raises here."""
        if isinstance(rows, (list, tuple)):
            # one [Hq, n_b] array per sequence; lengths may differ -> pad with NaN (the kernel
            # reads the pad as the end of the sequence's rows and checks it against valid_len)
            arrs = [np.asarray(x, dtype=np.float64) for x in rows]
            if len(arrs) != self.batch or any(a.ndim != 2 or a.shape[0] != self.shape.num_heads for a in arrs):
                raise ValueError(f"expected {self.batch} attention row blocks of shape [heads={self.shape.num_heads}, n]")
            lens = [a.shape[1] for a in arrs]
            ld = max(lens) + (1 if min(lens) != max(lens) else 0)
            pad = np.full((len(arrs), arrs[0].shape[0], max(ld, 1)), np.nan)
            for i, a in enumerate(arrs):
                pad[i, :, : a.shape[1]] = a
            r = torch.from_numpy(pad)
            sums = torch.from_numpy(np.stack([a.sum(axis=1) for a in arrs]))
        else:
            r = rows if isinstance(rows, torch.Tensor) else torch.as_tensor(np.asarray(rows, dtype=np.float64))
            if r.dim() == 2:
                r = r[None]
            if r.dim() != 3 or r.shape[0] != self.batch or r.shape[1] != self.shape.num_heads:
                raise ValueError(f"expected attention rows [batch={self.batch}, heads={self.shape.num_heads}, n]")
            sums = r.sum(dim=2)
        if torch.any((sums.double() - 1.0).abs() > 1e-4):
            raise ValueError(f"attention rows must each sum to 1 within 1e-4, got {sums}")
        with _on(stream):
            r = r.to(device=self.device, dtype=torch.float64).contiguous()
        _lib.check(self.lib.ckv_stage_rows(self._h, layer, _ptr(r), r.shape[2], _stream(stream)))
        self._rows_keep[layer] = r   # the staged tensor outlives the async launch (one per layer)

    def stage_weights(self, gathered, shards: int, layer_begin: int = 0, stream=None) -> None:
        """Head-sharded EMA input: `gathered` = every head shard's attention weights
        ([shards, layers, batch, Hq_local, capacity] fp32, shard order), summed over all
        heads in global head order (bit-identical to an unsharded engine)."""
        with _on(stream):
            g = gathered.to(device=self.device, dtype=torch.float32).contiguous()
        if g.dim() != 5 or g.shape[0] != shards or g.shape[2] != self.batch or g.shape[4] != self.capacity:
            raise ValueError(f"expected [shards={shards}, layers, {self.batch}, Hq_local, {self.capacity}]")
        _lib.check(self.lib.ckv_stage_weights(self._h, layer_begin, g.shape[1], _ptr(g), shards, _stream(stream)))
        self._stage_keep = g

    def head_partial(self, w, acc_in, acc_out, layer_begin: int = 0, stream=None) -> None:
        """Head-sharded chain step (ckv_head_partial): acc_out = acc_in (or 0) + this engine's
        heads' weights `w` ([layers, batch, Hq_local, capacity] fp32, from attend_layers) summed
        in head order in fp64; acc [layers, batch, capacity] fp64 (may alias)."""
        L = w.shape[0]
        for a in (acc_in, acc_out):
            if a is not None and (a.dtype != torch.float64 or tuple(a.shape) != (L, self.batch, self.capacity)
                                  or not a.is_contiguous()):
                raise ValueError(f"acc must be contiguous fp64 [{L}, {self.batch}, {self.capacity}]")
        _lib.check(self.lib.ckv_head_partial(self._h, layer_begin, L, _ptr(w), _ptr(acc_in), _ptr(acc_out),
                                             _stream(stream)))

    def stage_mass(self, acc, total_heads: int, layer_begin: int = 0, stream=None) -> None:
        """Stage head mean = acc / total_heads (the global head sums of the chain) for the
        next step (ckv_stage_mass)."""
        if acc.dtype != torch.float64 or acc.dim() != 3 or not acc.is_contiguous():
            raise ValueError("acc must be contiguous fp64 [layers, batch, capacity]")
        _lib.check(self.lib.ckv_stage_mass(self._h, layer_begin, acc.shape[0], _ptr(acc), int(total_heads),
                                           _stream(stream)))

    def _logits(self, logits, vocab):
        lg = logits if isinstance(logits, torch.Tensor) else torch.as_tensor(np.asarray(logits))
        if lg.dim() == 1:
            lg = lg[None]
        if lg.shape[0] != self.batch or lg.shape[1] < vocab:
            raise ValueError(f"expected logits [batch={self.batch}, V={vocab}], got {tuple(lg.shape)}")
        if lg.dtype not in (torch.float32, torch.bfloat16, torch.float64):
            lg = lg.to(torch.float32)
        lg = lg.to(self.device)
        if lg.stride(1) != 1:
            lg = lg.contiguous()
        return lg, _DTYPES[lg.dtype]

    def confidence(self, logits, stream=None) -> None:
        """K1 over full logits [batch, V] (confidence.py:31-87); features land in the records."""
        with _on(stream):
            lg, dt = self._logits(logits, self.shape.vocab_size)
        _lib.check(self.lib.ckv_confidence(self._h, _ptr(lg), dt, lg.stride(0), _stream(stream)))
        self._conf_keep = lg

    def confidence_partial(self, logits_slice, vocab_offset: int, stream=None) -> torch.Tensor:
        """This shard's online-softmax tuple ([batch, 8] fp64) over its logits slice
        (this engine's vocab_size columns starting at global id `vocab_offset`)."""
        with _on(stream):
            lg, dt = self._logits(logits_slice, self.shape.vocab_size)
        out = torch.empty((self.batch, 8), dtype=torch.float64, device=self.device)
        _lib.check(self.lib.ckv_confidence_partial(self._h, _ptr(lg), dt, lg.stride(0), int(vocab_offset),
                                                   _ptr(out), _stream(stream)))
        self._conf_keep = lg
        return out

    def confidence_merge(self, parts, vocab_total: int, stream=None) -> None:
        """Merge all shards' tuples ([shards, batch, 8] fp64, shard order) and finalise."""
        with _on(stream):
            p = parts.to(device=self.device, dtype=torch.float64).contiguous()
        _lib.check(self.lib.ckv_confidence_merge(self._h, _ptr(p), p.shape[0], int(vocab_total), _stream(stream)))
        self._merge_keep = p

    def manage(self, k_new, v_new, step: int, kept: bool = True, stream=None) -> StepResult:
        """ConfKVEngine._manage + append (policy.py:199-206, 256-274) after `confidence`
        (or the sharded merge) and attention/staging for every layer."""
        s = self.shape
        L, B = s.num_layers, self.batch
        with _on(stream):
            kn = self._half(k_new, (L, B, s.kv_heads, s.head_dim), "k_new")
            vn = self._half(v_new, (L, B, s.kv_heads, s.head_dim), "v_new")
        km, kl, vic = self._kept_bufs(kept)
        self._len_fresh = False
        self._pre_manage(int(step), stream)
        self._manage_launch(step, kn, vn, km, kl, vic, _stream(stream))
        self._keep = (kn, vn)
        self._last_step = int(step)
        self._next_t = int(step) + 1
        self.steps_run += 1
        return StepResult(None, km, kl, vic)

    # ------------------------------------------------------------------ step
    def step(self, logits, k_new, v_new, step: int, q=None, kept: bool = True, stream=None, out=None,
             attn_events=None):
        """DecodePolicy.step (policy.py:187-224) for every sequence.

        Two call forms. (1) The reference's own: `step(logits, attention_rows, new_kv, step)`
        with attention_rows[l] the [Hq, n] rows (one array per layer, or per layer a list of
        per-sequence arrays) and new_kv[l] = (k, v) [Hkv, D] -- stages the rows, runs the step,
        synchronises and returns the StepRecord (a list of them when batch > 1), exactly what
        `run_decode` consumes (simulator.py:468-476). (2) The device form:
        logits [batch, V] (fp32, bf16 or fp64, device or host); k_new/v_new
        [layers, batch, Hkv, D] fp16; q [layers, batch, Hq, D] computes the
        attention of every layer first (else `attend` must have run for each
        layer this step); K1 then runs on a side stream beside the attention and
        `attn_events` (two CUDA events, optional) bracket the attention on the
        step's stream. Asynchronous: returns a StepResult (outputs + kept-index map);
        use `records()` for the trace rows.
        """
        if isinstance(k_new, (list, tuple)) and q is None:
            recs = self.step_rows(logits, k_new, v_new, step, stream=stream)
            return recs[0] if self.batch == 1 else recs
        s = self.shape
        L, B = s.num_layers, self.batch
        with _on(stream):
            lg = logits if isinstance(logits, torch.Tensor) else torch.as_tensor(np.asarray(logits))
            if lg.dim() == 1:
                lg = lg[None]
            if lg.shape[0] != B or lg.shape[1] < s.vocab_size:
                raise ValueError(f"expected logits [batch={B}, V={s.vocab_size}], got {tuple(lg.shape)}")
            if lg.dtype not in (torch.float32, torch.bfloat16, torch.float64):
                lg = lg.to(torch.float32)
            lg = lg.to(self.device)
            if lg.stride(1) != 1:
                lg = lg.contiguous()
            kn = self._half(k_new, (L, B, s.kv_heads, s.head_dim), "k_new")
            vn = self._half(v_new, (L, B, s.kv_heads, s.head_dim), "v_new")
        dt = _DTYPES[lg.dtype]
        self._len_fresh = False
        km, kl, vic = self._kept_bufs(kept)
        st = _stream(stream)
        if q is not None:
            cur = stream if stream is not None else torch.cuda.current_stream(self.device)
            order = self._k1_order
            if order != "serial":
                # K1 reads only the logits: fork it onto the engine's side stream so it runs
                # beside K2 (the same fork/join ckv_step does for C callers); "after" forks it
                # once the attention grids are submitted, so it runs beside the combine
                if self._side is None:
                    self._side = torch.cuda.Stream(self.device)
                if order == "before":
                    self._side.wait_stream(cur)
                    _lib.check(self.lib.ckv_confidence(self._h, _ptr(lg), dt, lg.stride(0),
                                                       _stream(self._side)))
            if attn_events is not None:
                attn_events[0].record(cur)
            if order == "after":
                # K1 inline beside the tcgen05 grid when it fills the GPU, else on the side
                # stream beside the attention (ckv_attend_conf decides; same as ckv_step)
                out, _ = self.attend_layers(q, 0, cur, out=out, conf=(lg, dt, self._side))
            else:
                out, _ = self.attend_layers(q, 0, cur, out=out)
            if attn_events is not None:
                attn_events[1].record(cur)
            if order == "serial":
                _lib.check(self.lib.ckv_confidence(self._h, _ptr(lg), dt, lg.stride(0), st))
            else:
                cur.wait_stream(self._side)
            self._pre_manage(int(step), stream)
            self._manage_launch(step, kn, vn, km, kl, vic, st)
            self._keep = (lg, kn, vn)
        else:
            _lib.check(self.lib.ckv_confidence(self._h, _ptr(lg), dt, lg.stride(0), st))
            self._pre_manage(int(step), stream)
            self._manage_launch(step, kn, vn, km, kl, vic, st)
            self._keep = (lg, kn, vn)   # inputs must outlive the async launch
        self._last_step = int(step)
        self._next_t = int(step) + 1
        self.steps_run += 1
        return StepResult(out, km, kl, vic)

    def _kept_bufs(self, kept):
        """kept: False (no kept-index map), True (the engine's buffers), a (map [L, B, cap],
        len [L, B]) pair of int32 device tensors to write this step's map into, or a
        VictimList (the compact form). Returns (map, len, victims)."""
        if kept is False or kept is None:
            return None, None, None
        if kept is True:
            return self._kept_map, self._kept_len, None
        L, B = self.shape.num_layers, self.batch
        if isinstance(kept, VictimList):
            v = kept.buf
            if v.dtype != torch.int32 or tuple(v.shape) != (L, B, self.capacity) or not v.is_contiguous():
                raise ValueError(f"victim buffer must be contiguous int32 [{L}, {B}, {self.capacity}]")
            return None, None, v
        km, kl = kept
        if (km.dtype != torch.int32 or kl.dtype != torch.int32 or tuple(km.shape) != (L, B, self.capacity)
                or tuple(kl.shape) != (L, B) or not km.is_contiguous() or not kl.is_contiguous()):
            raise ValueError(f"kept buffers must be contiguous int32 [{L}, {B}, {self.capacity}] and [{L}, {B}]")
        return km, kl, None

    def _manage_launch(self, step, kn, vn, km, kl, vic, st):
        if vic is not None:
            _lib.check(self.lib.ckv_victims_out(self._h, _ptr(vic)))
        try:
            _lib.check(self.lib.ckv_manage(self._h, int(step), _ptr(kn), _ptr(vn), _ptr(km), _ptr(kl), st))
        finally:
            if vic is not None:
                self.lib.ckv_victims_out(self._h, None)

    def capture_step(self, logits, k_new, v_new, q, out=None, attn_events=None, after=None, before=None,
                     kept=True):
        """Capture one whole step — attention of every layer, K1 forked beside it, K3/K4 — as a
        CUDA graph over these (device, fixed-address) input tensors. Each `replay()` runs the
        engine's next step: the step counter lives on the device, so replays advance it
        without the host (which is what makes one launch per step possible for the small,
        launch-bound configs). `attn_events` must be created with `external=True` to be
        recorded inside the graph; `before(stream)` / `after(stream)` add work ahead of / after the
        step (e.g. the inputs' H2D copy, a records copy). Returns the torch.cuda.CUDAGraph; update the inputs in place between replays."""
        cur = torch.cuda.current_stream(self.device)
        # one capture stream per engine: torch hands out pool streams round-robin, so a fresh one
        # per capture would shift (and could alias) the streams later callers take from the pool
        if getattr(self, "_cap_side", None) is None:
            self._cap_side = torch.cuda.Stream(self.device)
        side = self._cap_side
        side.wait_stream(cur)
        # capture with the step number the library expects next, so no step-reset launch is
        # captured; several captures in a row get consecutive numbers (replay them in order)
        t = self._next_t
        last = self._last_step
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                if before is not None:
                    before(side)
                self.step(logits, k_new, v_new, step=t, q=q, kept=kept, stream=side, out=out,
                          attn_events=attn_events)
                if after is not None:
                    after(side)
        cur.wait_stream(side)
        # nothing ran during the capture: undo the host bookkeeping of the captured call
        self.steps_run -= 1
        self._last_step = last
        return g

    def note_replayed_steps(self, k: int) -> None:
        """Host bookkeeping after k replays of captured steps (records() then reports the last)."""
        self.steps_run += k
        self._len_fresh = False
        self._last_step = (self._last_step or 0) + k
        self._next_t = max(self._next_t, self._last_step + 1)

    def step_rows(self, logits, attention_rows, new_kv, step: int, stream=None) -> list[StepRecord]:
        """The reference's exact signature (policy.py:187-193) for batch 1 or
        batched inputs: attention_rows[l] [.., Hq, n] fp64, new_kv[l] = (k, v)
        [.., Hkv, D]. Returns the StepRecords (synchronises)."""
        L = self.shape.num_layers
        if len(attention_rows) != L or len(new_kv) != L:
            raise ValueError("attention_rows and new_kv must have one entry per layer")
        for layer, rows in enumerate(attention_rows):
            self.stage_rows(layer, rows, stream)
        ks = torch.stack([torch.as_tensor(np.asarray(k, dtype=np.float32)).reshape(self.batch, self.shape.kv_heads, -1)
                          for k, _ in new_kv])
        vs = torch.stack([torch.as_tensor(np.asarray(v, dtype=np.float32)).reshape(self.batch, self.shape.kv_heads, -1)
                          for _, v in new_kv])
        self.step(logits, ks, vs, step, stream=stream)
        return self.records(stream)

    # ------------------------------------------------------------------ outputs
    def records(self, stream=None) -> list[StepRecord]:
        """StepRecord per sequence for the last step (synchronises the stream)."""
        _lib.check(self.lib.ckv_read_records(self._h, C.cast(self._rec_l, C.c_void_p),
                                             C.cast(self._rec_s, C.c_void_p), _stream(stream)))
        recs = self._parse_records(self._rec_l, self._rec_s, self._last_step)
        if self._last_step is not None:
            lay = np.frombuffer(self._rec_l, dtype=_DT_LAYER, count=self.shape.num_layers * self.batch)
            self._host_len[:] = lay["len_after"].reshape(self.shape.num_layers, self.batch)
            self._len_fresh = True
        return recs

    def _parse_records(self, rec_l, rec_s, step: int) -> list[StepRecord]:
        """Device records (ctypes arrays / pinned buffers) -> StepRecords, vectorised over
        (layer, sequence) with NumPy (the per-step host cost of the pipelined e2e path)."""
        s, L, B = self.shape, self.shape.num_layers, self.batch
        if L * B < 96:
            return self._parse_records_loop(rec_l, rec_s, step)
        elems = s.kv_heads * s.head_dim
        lay = np.frombuffer(rec_l, dtype=_DT_LAYER, count=L * B).reshape(L, B)
        seq = np.frombuffer(rec_s, dtype=_DT_SEQ, count=B)
        status = np.bitwise_or.reduce(lay["status"], axis=0) | seq["status"]
        for st in status[status != 0].tolist():   # first failing sequence decides, as per-sequence checks would
            if st & _lib.ST_SHAPE:
                raise ValueError("attention rows must have exactly valid_len entries per head (cache.py:164-167)")
            if st & _lib.ST_NONFINITE:
                raise ValueError("logits must all be finite")
            if st & _lib.ST_NOATTEND:
                raise RuntimeError("step ran without attention rows for some layer")
            if st & _lib.ST_SCHEDULE:
                raise ValueError("schedule demands more evictions than there are candidates")
            if st & (_lib.ST_OVERFLOW | _lib.ST_SEGOVERFLOW):
                raise RuntimeError(f"cache capacity exhausted (status {st}); raise capacity/max_segments")
        n8 = lay["int8_count"].astype(np.int64)
        hi = lay["len_after"].astype(np.int64) - n8
        mem = ((hi * 2 + n8) * elems * 2 + lay["num_segments"].astype(np.int64) * 4 * elems * 2).sum(axis=0).tolist()
        len_pre, len_post = lay["len_pre"].T.tolist(), lay["len_post"].T.tolist()
        evicted, int8 = lay["evicted"].T.tolist(), n8.T.tolist()
        sc, en, mg = seq["score"].tolist(), seq["entropy_norm"].tolist(), seq["margin"].tolist()
        ms, tp = seq["margin_sig"].tolist(), seq["top_prob"].tolist()
        th, tok = seq["tier_high"].tolist(), seq["token"].tolist()
        out = []
        for b in range(B):
            if self.schedules is not None:
                for layer, ev in enumerate(evicted[b]):
                    if ev:
                        self.schedules[b].append(EvictionEvent(step, layer, ev))
            out.append(StepRecord(
                step=step, confidence=sc[b], entropy_norm=en[b], margin=mg[b], margin_sig=ms[b],
                top_prob=tp[b], budget=self._record_budget(_SeqTier(th[b])),
                len_pre=len_pre[b], len_post=len_post[b], evicted=evicted[b], int8=int8[b],
                memory_bytes=mem[b], token=tok[b]))
        return out

    def _parse_records_loop(self, rec_l, rec_s, step: int) -> list[StepRecord]:
        """Per-record ctypes reads: cheaper than NumPy below ~100 (layer, sequence) records."""
        s, L, B = self.shape, self.shape.num_layers, self.batch
        elems = s.kv_heads * s.head_dim
        out = []
        for b in range(B):
            sq = rec_s[b]
            lay = [rec_l[l * B + b] for l in range(L)]
            status = sq.status
            for r in lay:
                status |= r.status
            if status & _lib.ST_SHAPE:
                raise ValueError("attention rows must have exactly valid_len entries per head (cache.py:164-167)")
            if status & _lib.ST_NONFINITE:
                raise ValueError("logits must all be finite")
            if status & _lib.ST_NOATTEND:
                raise RuntimeError("step ran without attention rows for some layer")
            if status & _lib.ST_SCHEDULE:
                raise ValueError("schedule demands more evictions than there are candidates")
            if status & (_lib.ST_OVERFLOW | _lib.ST_SEGOVERFLOW):
                raise RuntimeError(f"cache capacity exhausted (status {status}); raise capacity/max_segments")
            mem = 0
            for r in lay:
                hi = r.len_after - r.int8_count
                mem += (hi * 2 + r.int8_count) * elems * 2 + r.num_segments * 4 * elems * 2
            tier = self._record_budget(sq)
            if self.schedules is not None:
                for layer, r in enumerate(lay):
                    if r.evicted:
                        self.schedules[b].append(EvictionEvent(step, layer, r.evicted))
            out.append(StepRecord(
                step=step, confidence=sq.score, entropy_norm=sq.entropy_norm,
                margin=sq.margin, margin_sig=sq.margin_sig, top_prob=sq.top_prob, budget=tier,
                len_pre=[r.len_pre for r in lay], len_post=[r.len_post for r in lay],
                evicted=[r.evicted for r in lay], int8=[r.int8_count for r in lay],
                memory_bytes=mem, token=sq.token))
        return out

    def _record_budget(self, sq):
        """StepRecord.budget: the tier (policy.py:260, 215)."""
        return self.config.n_high if sq.tier_high else self.config.n_low

    def _pre_manage(self, step: int, stream) -> None:
        """Hook run before every ckv_manage (the matched-rate replay uploads its counts)."""

    def read_cache(self, layer: int, seq: int = 0, stream=None) -> dict:
        """Host copy of one (layer, sequence) cache in the reference's
        LayerCache vocabulary (synchronises). Debug / parity only."""
        s = self.shape
        cap, row = self.capacity, s.kv_heads * s.head_dim
        n, nseg = C.c_int32(), C.c_int32()
        a = dict(positions=np.zeros(cap, np.int64), steps=np.zeros(cap, np.int64),
                 ema=np.zeros(cap, np.float64), seen=np.zeros(cap, np.uint8),
                 segment_of=np.zeros(cap, np.int32),
                 keys=np.zeros((cap, s.kv_heads, s.head_dim), np.float32),
                 values=np.zeros((cap, s.kv_heads, s.head_dim), np.float32),
                 k_codes=np.zeros((cap, s.kv_heads, s.head_dim), np.int8),
                 v_codes=np.zeros((cap, s.kv_heads, s.head_dim), np.int8))
        smax = cap
        sk = np.zeros((smax, s.kv_heads, s.head_dim), np.float32)
        sv = np.zeros_like(sk)
        sc = np.zeros(smax, np.int32)
        ptrs = [a[k].ctypes.data_as(C.c_void_p) for k in
                ("positions", "steps", "ema", "seen", "segment_of", "keys", "values", "k_codes", "v_codes")]
        _lib.check(self.lib.ckv_read_cache(self._h, layer, seq, C.byref(n), C.byref(nseg), *ptrs,
                                           sk.ctypes.data_as(C.c_void_p), sv.ctypes.data_as(C.c_void_p),
                                           sc.ctypes.data_as(C.c_void_p), _stream(stream)))
        m, g = n.value, nseg.value
        res = {k: v[:m] for k, v in a.items()}
        res["seen"] = res["seen"].astype(bool)
        res.update(valid_len=m, num_segments=g, seg_k_scale=sk[:g], seg_v_scale=sv[:g], seg_count=sc[:g])
        return res


_DT_LAYER = np.dtype(_lib.CkvLayerRecord)
_DT_SEQ = np.dtype(_lib.CkvSeqRecord)


class _SeqTier:
    """The one field of a sequence record `_record_budget` reads."""
    __slots__ = ("tier_high",)

    def __init__(self, tier_high: int):
        self.tier_high = tier_high


class HostPipeline:
    """Decode steps fed from host memory, pipelined (the drop-in for a host-side caller).

    ``submit`` enqueues one whole step for host-resident (pinned) inputs and returns at
    once: the inputs are copied H2D on a copy stream into one of ``depth`` device input
    sets while the previous step still computes; the step runs on the compute stream once
    its copy has landed; the attention output and the step's records go back D2H on a
    second copy stream into pinned buffers. Nothing synchronises until ``records(step)``
    or ``drain()``. Buffers are reused every ``depth`` steps, so a step's outputs are
    valid until step + depth is submitted.
    """

    def __init__(self, engine: "ConfKVEngine", depth: int = 2, stream=None, graphs: bool = False,
                 fused_copies: bool | None = None):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        # graphs=True: each input set's step (attention, K1, K3/K4, records copy) is captured once
        # as a CUDA graph and replayed (one launch per step; steps must then be consecutive)
        self.graphs = [None] * depth if graphs else None
        self._next = None
        e, s = engine, engine.shape
        dev = e.device
        self.engine, self.depth = e, depth
        self.compute = stream if stream is not None else torch.cuda.current_stream(dev)
        # copy streams from torch's high-priority pool: nothing else here takes from it, so they
        # never alias each other or a stream the step uses (the low-priority pool is round-robin)
        self.h2d = torch.cuda.Stream(dev, priority=-1)
        self.d2h = torch.cuda.Stream(dev, priority=-1)
        L, B = s.num_layers, e.batch
        self._shapes = dict(logits=((B, s.vocab_size), torch.float32), q=((L, B, s.num_heads, s.head_dim), torch.float16),
                            k=((L, B, s.kv_heads, s.head_dim), torch.float16),
                            v=((L, B, s.kv_heads, s.head_dim), torch.float16))
        # one device buffer per input set, each input a 256-byte-aligned view of it; host inputs
        # laid out the same way (`host_inputs()`) go H2D as one copy per step
        self._offs, off = {}, 0
        for k, (sh, dt) in self._shapes.items():
            self._offs[k] = off
            off += -(-int(np.prod(sh)) * torch.tensor([], dtype=dt).element_size() // 256) * 256
        self._packed_bytes = off
        self.packed_bytes = off                                     # H2D bytes per step via host_inputs()
        self._in_buf = [torch.empty(off, dtype=torch.uint8, device=dev) for _ in range(depth)]
        self._in = [self._views(buf) for buf in self._in_buf]
        self._out = [torch.empty((L, B, s.num_heads, s.head_dim), dtype=torch.float32, device=dev)
                     for _ in range(depth)]
        # the step's kept-index map (north star: step -> attention output + kept-index map) in
        # compact form: K3 writes each cache's evicted indices into the input set's device
        # buffer; the first `vmax` per cache go D2H with the records (a cache that evicted
        # more -- a tier switch, step 1 -- is fetched by kept() from the set's buffer)
        cap = e.capacity
        self.vmax = 4
        self._vic = [torch.empty((L, B, cap), dtype=torch.int32, device=dev) for _ in range(depth)]
        nl, ns = C.sizeof(_lib.CkvLayerRecord) * L * B, C.sizeof(_lib.CkvSeqRecord) * B
        # a step's records + leading victims are packed on the device into one block per set
        # (ckv_pack_outputs, inside the step) and go D2H as one copy beside the next step
        self._nwords = (nl + ns) // 4 + L * B * self.vmax
        self._stage_dev = [torch.empty(self._nwords, dtype=torch.int32, device=dev) for _ in range(depth)]
        self._stage_host = [torch.empty(self._nwords, dtype=torch.int32).pin_memory() for _ in range(depth)]
        self._rec = [(h.data_ptr(), h.data_ptr() + nl) for h in self._stage_host]   # record addresses
        self._vic_host = [h[(nl + ns) // 4:].view(L, B, self.vmax) for h in self._stage_host]
        self._ev_in = [torch.cuda.Event() for _ in range(depth)]     # H2D of set i landed
        self._ev_done = [torch.cuda.Event() for _ in range(depth)]   # step using set i finished
        self._ev_out = [torch.cuda.Event() for _ in range(depth)]    # D2H of set i finished
        self._steps = [None] * depth
        self.h2d_bytes = sum(int(np.prod(sh)) * torch.tensor([], dtype=dt).element_size()
                             for sh, dt in self._shapes.values())
        self.d2h_bytes = self._out[0].numel() * 4 + nl + ns + L * B * self.vmax * 4
        # fused_copies (graphs only): a step's H2D input copy and D2H output copy are captured
        # into its graph — one launch per step, copies serialised with compute. Pays off when the
        # per-step host work outweighs the copies (small, launch-bound configs); default: when a
        # step moves <= 512 KB. Needs host_inputs() buffers, the same ones per input set.
        # (r02: the steady state of the overlapped path is one C call per step, ckv_pipe_submit,
        # which beats fusing: GPT-2 shape, batch 1: 67 -> see profiles/README.md us per e2e step)
        if fused_copies is None:
            fused_copies = False
        self.fused = bool(fused_copies) and self.graphs is not None
        self._gkeys = [None] * depth
        # host-side fast path: the (logits, q, k, v, out) pointers a set last validated with, and
        # the packed view of host_inputs() buffers (building it costs more than a small step)
        self._valid = [None] * depth
        self._handles = [None] * depth
        self._csubmit = os.environ.get("CKV_CSUBMIT", "1") != "0"
        self.c_submits = 0                  # steps submitted through ckv_pipe_submit
        self._packed = {}
        # numpy views of the pinned record / victim buffers (kept() reads them every step)
        self._rec_np = [(h[:nl // 4].numpy().reshape(L, B, 8), h[nl // 4:(nl + ns) // 4].numpy().reshape(B, 14))
                        for h in self._stage_host]
        self._vic_np = [v.numpy() for v in self._vic_host]

    def _views(self, buf):
        out = {}
        for k, (sh, dt) in self._shapes.items():
            nb = int(np.prod(sh)) * torch.tensor([], dtype=dt).element_size()
            out[k] = buf[self._offs[k]:self._offs[k] + nb].view(dt).view(sh)
        return out

    def host_inputs(self) -> dict:
        """Pinned host tensors (logits, q, k, v) laid out like the device input sets: fill them
        and pass them to `submit`, and the step's inputs go H2D as one copy."""
        buf = torch.empty(self._packed_bytes, dtype=torch.uint8).pin_memory()
        d = self._views(buf)
        d["_buf"] = buf
        return d

    def _packed_source(self, src):
        base = src["logits"]
        try:
            p0 = base.data_ptr() - self._offs["logits"]
            if not all(src[k].is_contiguous() and src[k].data_ptr() == p0 + self._offs[k] for k in self._shapes):
                return None
            st = base.untyped_storage()
            if st.data_ptr() > p0 or p0 + self._packed_bytes > st.data_ptr() + st.nbytes():
                return None
        except RuntimeError:
            return None
        return torch.empty(0, dtype=torch.uint8).set_(st, p0 - st.data_ptr(), (self._packed_bytes,))

    def submit(self, step: int, logits, q, k_new, v_new, out=None) -> None:
        """Enqueue decode step `step` from host tensors (pinned for overlap); `out`
        (optional, pinned fp32 [layers, batch, Hq, D]) receives the attention output."""
        i = step % self.depth
        key = (logits.data_ptr(), q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(),
               0 if out is None else out.data_ptr())
        if self.fused and self._valid[i] == key and step == self._next:
            # the same validated host buffers as this set's captured graph: replay directly
            with torch.cuda.stream(self.compute):
                self.graphs[i].replay()
                self._ev_done[i].record(self.compute)
                self._ev_out[i].record(self.compute)
            self.engine.note_replayed_steps(1)
            self._next = step + 1
            self._steps[i] = step
            return
        if (self._csubmit and not self.fused and self.graphs is not None and self._valid[i] == key
                and step == self._next and self.graphs[i] is not None):
            # steady state, overlapped copies: H2D of this set, the step's graph, D2H of its output
            # -- one C call (ckv_pipe_submit) instead of a dozen runtime calls from Python
            h = self._handles[i]
            _lib.check(self.engine.lib.ckv_pipe_submit(
                h[0], h[1], h[2], h[3], h[4], C.c_void_p(self._packed[key[:4]].data_ptr()), self._packed_bytes,
                h[5], h[6], h[7], 0, C.c_void_p(key[4]) if key[4] else None, h[8], h[9], h[10], h[11], h[12]))
            self.engine.note_replayed_steps(1)
            self._next = step + 1
            self._steps[i] = step
            self.c_submits += 1
            return
        src = dict(logits=logits, q=q, k=k_new, v=v_new)
        for k, (sh, dt) in self._shapes.items():
            t = src[k]
            if tuple(t.shape) != sh or t.dtype != dt:
                raise ValueError(f"{k}: expected {dt} {sh}, got {t.dtype} {tuple(t.shape)}")
        dst = self._in[i]
        # a graph freezes the launch plan of the step it was captured at; the engine's first
        # step (nothing demoted yet: every split on the general kernel) runs eagerly
        use_graph = self.graphs is not None and step >= 2
        if self.fused and use_graph:
            packed = self._packed.get(key[:4])
            if packed is None:
                packed = self._packed_source(src)
                if packed is not None:
                    self._packed[key[:4]] = packed
            if packed is not None:
                self._submit_fused(step, i, packed, out)
                self._valid[i] = key
                return
        with torch.cuda.stream(self.h2d):
            if self._steps[i] is not None:
                self.h2d.wait_event(self._ev_done[i])   # set i no longer read by step - depth
            packed = self._packed.get(key[:4])
            if packed is None:
                packed = self._packed_source(src)
                if packed is not None:
                    self._packed[key[:4]] = packed
            if packed is not None:                      # `host_inputs()` layout: one copy
                self._in_buf[i].copy_(packed, non_blocking=True)
            else:
                for k in dst:
                    dst[k].copy_(src[k], non_blocking=True)
            self._ev_in[i].record(self.h2d)
        self.compute.wait_event(self._ev_in[i])
        if self._steps[i] is not None:
            self.compute.wait_event(self._ev_out[i])    # out[i] of step - depth copied out
        e = self.engine

        def copy_records(st):   # (device side: the D2H copy runs on the d2h stream below)
            _lib.check(e.lib.ckv_pack_outputs(e._h, C.c_void_p(self._stage_dev[i].data_ptr()),
                                              C.c_void_p(self._vic[i].data_ptr()), self.vmax, _stream(st)))

        with torch.cuda.stream(self.compute):
            if use_graph:
                if self._next is not None and step != self._next:
                    raise ValueError(f"graph pipeline needs consecutive steps (expected {self._next}, got {step})")
                if self.graphs[i] is None:
                    if step != e._next_t:
                        raise ValueError(f"step {step} is not the engine's next step {e._next_t}")
                    self.graphs[i] = e.capture_step(dst["logits"], dst["k"], dst["v"], dst["q"],
                                                    out=self._out[i], after=copy_records,
                                                    kept=VictimList(self._vic[i]))
                self.graphs[i].replay()
                e.note_replayed_steps(1)
                self._next = step + 1
            else:
                e.step(dst["logits"], dst["k"], dst["v"], step=step, q=dst["q"], kept=VictimList(self._vic[i]),
                       stream=self.compute, out=self._out[i])
                copy_records(self.compute)
                if self.graphs is not None:
                    self._next = step + 1
            self._ev_done[i].record(self.compute)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self._ev_done[i])
            if out is not None:
                out.copy_(self._out[i], non_blocking=True)
            self._stage_host[i].copy_(self._stage_dev[i], non_blocking=True)
            self._ev_out[i].record(self.d2h)
        self._steps[i] = step
        if use_graph and packed is not None and (out is None or (out.is_pinned() and out.is_contiguous())):
            # this set's raw handles for ckv_pipe_submit (the events now exist: recorded above)
            self._handles[i] = (
                C.c_void_p(self.graphs[i].raw_cuda_graph_exec()), C.c_void_p(self.compute.cuda_stream),
                C.c_void_p(self.h2d.cuda_stream), C.c_void_p(self.d2h.cuda_stream),
                C.c_void_p(self._in_buf[i].data_ptr()), C.c_void_p(self._ev_in[i].cuda_event),
                C.c_void_p(self._ev_done[i].cuda_event), C.c_void_p(self._ev_out[i].cuda_event),
                C.c_void_p(self._out[i].data_ptr()), self._out[i].numel() * 4,
                C.c_void_p(self._stage_host[i].data_ptr()), C.c_void_p(self._stage_dev[i].data_ptr()),
                self._nwords * 4)
            self._valid[i] = key

    def _submit_fused(self, step, i, packed, out) -> None:
        e = self.engine
        key = (packed.data_ptr(), 0 if out is None else out.data_ptr())
        if self.graphs[i] is None:
            if self._next is not None and step != self._next:
                raise ValueError(f"graph pipeline needs consecutive steps (expected {self._next}, got {step})")
            if step != e._next_t:
                raise ValueError(f"step {step} is not the engine's next step {e._next_t}")
            dst, o = self._in[i], self._out[i]

            def before(st):
                self._in_buf[i].copy_(packed, non_blocking=True)

            def after(st):
                _lib.check(e.lib.ckv_pack_outputs(e._h, C.c_void_p(self._stage_dev[i].data_ptr()),
                                                  C.c_void_p(self._vic[i].data_ptr()), self.vmax, _stream(st)))
                self._stage_host[i].copy_(self._stage_dev[i], non_blocking=True)
                if out is not None:
                    out.copy_(o, non_blocking=True)

            with torch.cuda.stream(self.compute):
                self.graphs[i] = e.capture_step(dst["logits"], dst["k"], dst["v"], dst["q"], out=o,
                                                before=before, after=after, kept=VictimList(self._vic[i]))
            self._gkeys[i] = key
        elif self._gkeys[i] != key:
            raise ValueError("fused-copy pipeline: pass the same host_inputs() / out buffers for an input set")
        elif step != self._next:
            raise ValueError(f"graph pipeline needs consecutive steps (expected {self._next}, got {step})")
        with torch.cuda.stream(self.compute):
            self.graphs[i].replay()
            self._ev_done[i].record(self.compute)
            self._ev_out[i].record(self.compute)
        e.note_replayed_steps(1)
        self._next = step + 1
        self._steps[i] = step

    def records(self, step: int) -> list[StepRecord]:
        """StepRecords of a submitted step still in the window (waits for that step only)."""
        i = step % self.depth
        if self._steps[i] != step:
            raise ValueError(f"step {step} is not in the pipeline window")
        self._ev_out[i].synchronize()                   # the step's packed outputs are on the host
        rl, rs = self._rec[i]
        L, B = self.engine.shape.num_layers, self.engine.batch
        lay = (_lib.CkvLayerRecord * (L * B)).from_address(rl)
        seq = (_lib.CkvSeqRecord * B).from_address(rs)
        return self.engine._parse_records(lay, seq, step)

    def kept(self, step: int) -> KeptMaps:
        """The kept-index maps of a submitted step still in the window (waits for that step):
        kept[l][b] = the pre-step storage indices of the survivors, in order (policy.py:117-127,
        cache.py:206), held as the step's victim lists + pre-step lengths (KeptMaps). Raises like
        records() when a record carries an error status."""
        i = step % self.depth
        if self._steps[i] != step:
            raise ValueError(f"step {step} is not in the pipeline window")
        self._ev_out[i].synchronize()                   # the step's packed outputs are on the host
        lay, seq = self._rec_np[i]
        if lay[:, :, 6].any() or seq[:, 12].any():
            self.records(step)                        # raises the record's error
        ev = lay[:, :, 2].copy()
        over = {}
        if ev.max() > self.vmax:
            for layer, b in zip(*np.nonzero(ev > self.vmax)):
                over[(int(layer), int(b))] = self._vic[i][layer, b, :ev[layer, b]].cpu().numpy()
        return KeptMaps(lay[:, :, 0].copy(), ev, self._vic_np[i].copy(), over)

    def drain(self) -> None:
        """Wait for every submitted step and copy."""
        for ev in self._ev_out + self._ev_done:
            ev.synchronize()


__all__ = ["ConfKVEngine", "HostPipeline", "StepRecord", "StepResult", "EvictionEvent", "ConfigError",
           "LayerCacheView", "VictimList", "kept_from_victims"]
