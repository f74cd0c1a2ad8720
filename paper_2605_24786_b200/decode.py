"""Decode loop on B200: the reference's seeded decoder stack driving the Conf-KV engine
(SURVEY §8 F1).

`DecodeModel` restates `ReferenceModel` (reference `simulator.py:29-92`): a token
embedding, per layer Q/K/V/O projections with a residual add, and a vocabulary
projection scaled by `logit_gain`; no MLP, no normalisation. The one extension is GQA
(`w_k`/`w_v` project to `num_kv_heads * head_dim`), as for the engine. The projections
are plain library GEMMs (cuBLAS through torch, bf16 by default, fp32 for parity runs);
the attention of every layer is `ConfKVEngine.attend_layers` (K2, the hot path), the
policy step is `ConfKVEngine.step` (K1 + K3/K4), and the next token comes from K1's
device-side greedy argmax (`ckv_tokens`) — one decode step never touches the host, so
it is captured once and replayed as a CUDA graph.

`run_decode` mirrors `simulator.run_decode` + `ModelDriver` (simulator.py:379-478):
token-by-token prefill through the model forward, then `steps` decode steps starting
from the last prompt token (the reference re-feeds it at step 1, simulator.py:401-402),
one `StepRecord` per step and sequence.
"""

from __future__ import annotations

import ctypes as C
import json
import math

import torch

from . import _lib
from .config import ModelShape
from .engine import ConfKVEngine, StepRecord


class DecodeModel:
    """ReferenceModel (simulator.py:29-92) on the device, batched over sequences.

    Weights: either `weights` (a dict with the reference's names — `embedding` [V, d],
    `w_q` [L, d, Hq*D], `w_k`/`w_v` [L, d, Hkv*D], `w_o` [L, Hq*D, d], `w_out` [d, V] —
    e.g. a reference model's arrays for a parity run) or seeded N(0,1) draws scaled as
    the reference scales them (1/sqrt(d); `w_out` also by `logit_gain`).
    """

    def __init__(self, shape: ModelShape, seed: int = 0, logit_gain: float = 8.0,
                 dtype: torch.dtype = torch.bfloat16, device=None, weights: dict | None = None):
        if shape.vocab_size < 1:
            raise ValueError("empty vocabulary")
        self.shape, self.seed, self.logit_gain, self.dtype = shape, seed, logit_gain, dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        L, Hq, Hkv, D, V = shape.num_layers, shape.num_heads, shape.kv_heads, shape.head_dim, shape.vocab_size
        d, kvd = Hq * D, Hkv * D
        self.d_model, self.kv_dim = d, kvd
        dev = self.device
        if weights is None:
            g = torch.Generator(device=dev)
            g.manual_seed(int(seed))
            scale = 1.0 / math.sqrt(d)

            def mat(*sz, s=1.0):
                return (torch.randn(sz, generator=g, device=dev, dtype=torch.float32) * s).to(dtype)

            self.embedding = mat(V, d)
            self.w_qkv = torch.cat([mat(L, d, d, s=scale), mat(L, d, kvd, s=scale), mat(L, d, kvd, s=scale)], dim=2)
            self.w_o = mat(L, d, d, s=scale)
            self.w_out = mat(d, V, s=scale * logit_gain)
        else:
            def t(x):
                return torch.as_tensor(x).to(device=dev, dtype=dtype).contiguous()

            self.embedding = t(weights["embedding"])
            wq = torch.as_tensor(weights["w_q"])
            wk = torch.as_tensor(weights["w_k"])
            wv = torch.as_tensor(weights["w_v"])
            if tuple(wq.shape) != (L, d, d) or tuple(wk.shape) != (L, d, kvd) or tuple(wv.shape) != (L, d, kvd):
                raise ValueError("projection weights do not match the shape")
            self.w_qkv = t(torch.cat([wq, wk, wv], dim=2))
            self.w_o = t(weights["w_o"])
            self.w_out = t(weights["w_out"])
        if tuple(self.embedding.shape) != (V, d) or tuple(self.w_out.shape) != (d, V):
            raise ValueError("embedding / output projection do not match the shape")

    @property
    def weight_bytes_per_step(self) -> int:
        """Bytes of weights one decode step streams (every projection once)."""
        es = self.w_qkv.element_size()
        return (self.w_qkv.numel() + self.w_o.numel() + self.w_out.numel()) * es

    def forward(self, engine: ConfKVEngine, tokens: torch.Tensor, q_buf: torch.Tensor, k_buf: torch.Tensor,
                v_buf: torch.Tensor, attn_out: torch.Tensor, stream=None) -> torch.Tensor:
        """One decode forward for every sequence over the engine's current caches
        (simulator.py:58-92). tokens: [B] int device; q_buf/k_buf/v_buf: fp16
        [L, B, H*, D] (this step's q and new K/V, written here); attn_out: fp32
        [L, B, Hq, D]. Returns the logits [B, V] fp32. Does not mutate the caches."""
        s = self.shape
        L, B = s.num_layers, tokens.shape[0]
        d, kvd = self.d_model, self.kv_dim
        x = self.embedding.index_select(0, tokens).float()   # fp32 residual stream
        bf16 = self.dtype == torch.bfloat16
        st = C.c_void_p((stream if stream is not None else torch.cuda.current_stream()).cuda_stream)
        for layer in range(L):
            qkv = torch.matmul(x.to(self.dtype), self.w_qkv[layer])
            if bf16:   # one fused split + fp16 conversion (decode_glue.cu)
                _lib.check(engine.lib.ckv_qkv_split(C.c_void_p(qkv.data_ptr()), B, d, kvd,
                                                    C.c_void_p(q_buf[layer].data_ptr()),
                                                    C.c_void_p(k_buf[layer].data_ptr()),
                                                    C.c_void_p(v_buf[layer].data_ptr()), st))
            else:
                q_buf[layer].copy_(qkv[:, :d].view(B, s.num_heads, s.head_dim))
                k_buf[layer].copy_(qkv[:, d:d + kvd].view(B, s.kv_heads, s.head_dim))
                v_buf[layer].copy_(qkv[:, d + kvd:].view(B, s.kv_heads, s.head_dim))
            engine.attend_layers(q_buf[layer:layer + 1], layer, stream, out=attn_out[layer:layer + 1])
            # empty caches contribute nothing (simulator.py:84-90): K2 returns zeros for n = 0
            o = attn_out[layer].reshape(B, d).to(self.dtype)
            if bf16:   # residual add in the GEMM epilogue, fp32 out
                x = torch.addmm(x, o, self.w_o[layer], out_dtype=torch.float32)
            else:
                x = x + torch.matmul(o, self.w_o[layer])
        if bf16:
            return torch.mm(x.to(self.dtype), self.w_out, out_dtype=torch.float32)
        return torch.matmul(x, self.w_out)


class DecodeLoop:
    """Batched greedy decode of `DecodeModel` through a `ConfKVEngine`, one CUDA graph per step.

    The step is: forward (per layer: QKV GEMM, K2 attention over the pre-step cache, O GEMM +
    residual), logits GEMM, then the policy step (K1 confidence + greedy token, K3 manage, K4
    demotion + append of this step's K/V) and the device-side token feedback.
    """

    def __init__(self, engine: ConfKVEngine, model: DecodeModel, use_graph: bool = True):
        s = engine.shape
        if model.shape != s:
            raise ValueError("model and engine shapes differ")
        self.engine, self.model, self.use_graph = engine, model, use_graph
        L, B, dev = s.num_layers, engine.batch, engine.device
        self.tokens = torch.zeros(B, dtype=torch.int32, device=dev)
        self.q = torch.empty((L, B, s.num_heads, s.head_dim), dtype=torch.float16, device=dev)
        self.k = torch.empty((L, B, s.kv_heads, s.head_dim), dtype=torch.float16, device=dev)
        self.v = torch.empty_like(self.k)
        self.attn = torch.zeros((L, B, s.num_heads, s.head_dim), dtype=torch.float32, device=dev)
        self.logits = torch.empty((B, s.vocab_size), dtype=torch.float32, device=dev)
        self.graph = None
        self.t = 0

    def _body(self, step: int, stream) -> None:
        e = self.engine
        lg = self.model.forward(e, self.tokens, self.q, self.k, self.v, self.attn, stream)
        self.logits.copy_(lg)
        e.step(self.logits, self.k, self.v, step=step, kept=False, stream=stream)
        _lib.check(e.lib.ckv_tokens(e._h, C.c_void_p(self.tokens.data_ptr()), C.c_void_p(stream.cuda_stream)))

    def prefill(self, prompt: torch.Tensor) -> None:
        """ModelDriver.prefill (simulator.py:395-399): every prompt token runs the forward
        over the cache built so far and appends its K/V (append_prefill) at its position.
        prompt: [B, P] token ids (host or device)."""
        e = self.engine
        prompt = torch.as_tensor(prompt).to(e.device, torch.int32)
        B, P = prompt.shape
        if B != e.batch or P < 1:
            raise ValueError("model driver needs at least one prompt token per sequence")
        e.begin_prefill(P)
        stream = torch.cuda.current_stream(e.device)
        for pos in range(P):
            self.tokens.copy_(prompt[:, pos])
            self.model.forward(e, self.tokens, self.q, self.k, self.v, self.attn, stream)
            e.prefill(self.k[:, :, None], self.v[:, :, None], first_pos=pos, stream=stream)
        self.tokens.copy_(prompt[:, -1])   # first_token(): the last prompt token is re-fed
        self.t = 0

    def step(self) -> None:
        """One decode step for every sequence (asynchronous; graph-replayed after the first)."""
        self.t += 1
        stream = torch.cuda.current_stream(self.engine.device)
        if not self.use_graph:
            self._body(self.t, stream)
            return
        if self.graph is None:
            # the first step runs eagerly (allocator warm-up), the second is captured; the
            # engine's step counter lives on the device, so replays advance it by themselves
            if self.t == 1:
                self._body(self.t, stream)
                return
            side = torch.cuda.Stream(self.engine.device)
            side.wait_stream(stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    self._body(self.t, side)
            stream.wait_stream(side)
            self.graph = g
        self.graph.replay()

    def records(self) -> list[StepRecord]:
        """StepRecords of the last step (synchronises)."""
        recs = self.engine.records()
        for r in recs:
            r.step = self.t
        return recs


def run_decode(engine: ConfKVEngine, model: DecodeModel, prompt, steps: int, sink=None,
               use_graph: bool = True) -> list[list[StepRecord]]:
    """simulator.run_decode (simulator.py:448-478) with the model driver, for every sequence:
    prefill, then `steps` greedy decode steps; returns records[t][b] and writes each as a
    JSONL line ({"seq": b, **StepRecord.to_dict()}) to `sink` when given."""
    loop = DecodeLoop(engine, model, use_graph=use_graph)
    loop.prefill(prompt)
    out = []
    for _ in range(steps):
        loop.step()
        recs = loop.records()
        out.append(recs)
        if sink is not None:
            for b, r in enumerate(recs):
                sink.write(json.dumps({"seq": b, **r.to_dict()}) + "\n")
    return out


__all__ = ["DecodeModel", "DecodeLoop", "run_decode"]
