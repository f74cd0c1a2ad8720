"""Multi-GPU layouts of the cache manager, one process per GPU.

* Sequence sharding (configs C5): sequences are independent engines in the reference
  (`policy.py:147-161`), so rank r simply owns the contiguous batch slice
  `shard_range(total, world, r)`; no collective on the data path. `bench.py` uses it.
* Head sharding (config C3): rank r owns KV heads [r*Hkv/W, (r+1)*Hkv/W) and their query
  heads, for every layer and sequence. Attention, INT8 scales (per head and channel,
  `quantizer.py:28`) and K/V storage are local; the kept set is per layer and the EMA is
  the mean over ALL heads (`cache.py:171`), a sequential fp64 sum in head order. Default
  exchange ("chain"): rank r receives rank r-1's running fp64 head sums, adds its own heads
  in order (`ckv_head_partial`) and passes them on; the last rank broadcasts the full sums
  and every rank stages sum / Hq (`ckv_stage_mass`) -- bit-identical to one GPU, hence
  identical kept sets, codes and records on every rank, at L*B*cap*8 bytes per hop (plus one
  broadcast) instead of every head's fp32 weights. "gather" all-gathers the weights instead
  (`ckv_stage_weights`; one collective, Hq/2 x the bytes).
* Vocab-sharded confidence: each rank reduces its logits slice to one online-softmax
  tuple per sequence (`ckv_confidence_partial`); the tuples are all-gathered and merged in
  rank order (`ckv_confidence_merge`).

Collectives go through `torch.distributed` (NCCL over NVLink on the GPU box; gloo in the
CPU tests). The exchange helpers take any process group, so they are tested on CPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) of `total` units for `rank` of `world` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    q, r = divmod(total, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def _host_staged(t: torch.Tensor, group=None) -> bool:
    """gloo moves host memory only: device tensors are staged through the host (the multi-rank
    harness on one GPU; NCCL takes device tensors directly)."""
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_gather_stack(t: torch.Tensor, group=None) -> torch.Tensor:
    """[world, *t.shape] with rank r's tensor at index r (shard order)."""
    world = dist.get_world_size(group)
    flat = t.contiguous().reshape(-1)
    staged = _host_staged(flat, group)
    src = flat.cpu() if staged else flat
    out = torch.empty((world * flat.numel(),), dtype=t.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)   # concatenated form (NCCL and gloo)
    return out.to(t.device).view(world, *t.shape)


def max_over_ranks(x: float, device, group=None) -> float:
    t = torch.tensor([x], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def head_mean_global(gathered: torch.Tensor) -> torch.Tensor:
    """Host restatement of `k2_stage_weights`: gathered [W, L, B, Hq_local, n] -> mean over
    all W*Hq_local heads, summed sequentially in global head order in fp64."""
    w = gathered.to(torch.float64)
    W, L, B, H, n = w.shape
    acc = torch.zeros((L, B, n), dtype=torch.float64, device=w.device)
    for r in range(W):
        for g in range(H):
            acc = acc + w[r, :, :, g]
    return acc / float(W * H)


def chain_head_sums(partial, acc: torch.Tensor, group=None) -> torch.Tensor:
    """Global-head-order fp64 head sums over the ranks of `group`, in place in `acc`
    ([L, B, cap] fp64, same shape on every rank): rank 0 starts the chain, rank r waits for
    rank r-1's sums, `partial(acc_in_or_None, acc)` adds its own heads in order, rank r hands
    them to r+1; the last rank's sums are broadcast to all. Returns acc."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    glob = (lambda r: r) if group is None else (lambda r: dist.get_global_rank(group, r))
    host = torch.empty(acc.shape, dtype=acc.dtype) if _host_staged(acc, group) else None
    wire = acc if host is None else host
    if rank > 0:
        dist.recv(wire, src=glob(rank - 1), group=group)
        if host is not None:
            acc.copy_(host)
    partial(acc if rank > 0 else None, acc)
    if host is not None:
        host.copy_(acc)
    if rank < world - 1:
        dist.send(wire, dst=glob(rank + 1), group=group)
    dist.broadcast(wire, src=glob(world - 1), group=group)
    if host is not None:
        acc.copy_(host)
    return acc


def chain_bytes_per_rank(L: int, B: int, cap: int, world: int) -> int:
    """Bytes one rank receives per step in the chain exchange (one hop + the broadcast)."""
    return 0 if world <= 1 else 2 * L * B * cap * 8


def gather_bytes_per_rank(L: int, B: int, hq_local: int, cap: int, world: int) -> int:
    """Bytes one rank receives per step when all-gathering every head's fp32 weights."""
    return (world - 1) * L * B * hq_local * cap * 4


class HeadShardedStep:
    """Drives one rank's head-sharded `ConfKVEngine` through a decode step.

    The engine must be built with this rank's head slice:
    `ModelShape(L, Hq // W, D, V, num_kv_heads=Hkv // W)`. Logits are either the full
    vocabulary (replicated on every rank) or this rank's vocab slice.
    """

    def __init__(self, engine, group=None, vocab_total: int | None = None, vocab_offset: int = 0,
                 exchange: str = "chain"):
        if exchange not in ("chain", "gather"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.eng = engine
        self.group = group
        self.world = dist.get_world_size(group)
        self.vocab_total = vocab_total
        self.vocab_offset = vocab_offset
        self.exchange = exchange
        s = engine.shape
        self._acc = torch.empty((s.num_layers, engine.batch, engine.capacity), dtype=torch.float64,
                                device=engine.device)
        self._w = torch.zeros((s.num_layers, engine.batch, s.num_heads, engine.capacity), dtype=torch.float32,
                              device=engine.device)
        self._out = torch.empty((s.num_layers, engine.batch, s.num_heads, s.head_dim), dtype=torch.float32,
                                device=engine.device)
        L, B, cap = s.num_layers, engine.batch, engine.capacity
        self.bytes_per_step = (chain_bytes_per_rank(L, B, cap, self.world) if exchange == "chain"
                               else gather_bytes_per_rank(L, B, s.num_heads, cap, self.world))

    def step(self, logits, q_local, k_local, v_local, step: int, kept=True, attn_events=None):
        eng = self.eng
        cur = torch.cuda.current_stream(eng.device)
        if attn_events is not None:
            attn_events[0].record(cur)
        out, w = eng.attend_layers(q_local, weights=self._w, out=self._out)
        if attn_events is not None:
            attn_events[1].record(cur)
        if self.exchange == "chain":
            chain_head_sums(lambda acc_in, acc_out: eng.head_partial(w, acc_in, acc_out), self._acc, self.group)
            eng.stage_mass(self._acc, self.world * eng.shape.num_heads)
        else:
            eng.stage_weights(all_gather_stack(w, self.group), self.world)
        if self.vocab_total is None:
            eng.confidence(logits)
        else:
            part = eng.confidence_partial(logits, self.vocab_offset)
            eng.confidence_merge(all_gather_stack(part, self.group), self.vocab_total)
        res = eng.manage(k_local, v_local, step, kept=kept)
        res.out = out
        return res
