"""Trace and snapshot I/O for GPU runs, in the reference's formats so a
GPU run diffs against the CPU reference's outputs.

- StepRecord JSONL: one `json.dumps(record.to_dict())` line per step, the schema and key
  order of `StepRecord.to_dict` (reference policy.py:54-69) and the sink protocol of
  `run_decode` (simulator.py:471-472). Batched engines write one file per sequence.
- `summarize_trace`: the deterministic aggregates of analysis.py:189-208 (`TraceSummary`,
  analysis.py:165-186), host-side over the records.
- CKVS snapshots: `LayerCache.write_snapshot` / `read_snapshot` (cache.py:278-326) — magic
  "CKVS", little-endian u32 layer_id, valid_len, heads, head_dim, then K and V as float32
  [valid_len, heads, head_dim] (the dequantized view: INT8 entries as code * scale), positions
  and steps int64, EMA float64, seen u8 — written from one (layer, sequence) cache of the
  device state. heads = the engine's KV heads (the reference is MHA-only; for GQA its
  expanded cache would repeat each KV head over its group).
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass

import numpy as np

from .engine import StepRecord

_SNAP_MAGIC = b"CKVS"


def write_jsonl(records, sink) -> None:
    """Append StepRecords to an open text sink, one JSON object per line."""
    for r in records:
        sink.write(json.dumps(r.to_dict()) + "\n")


def read_jsonl(path) -> list[StepRecord]:
    out = []
    with open(path) as f:
        for line in f:
            if line.strip():
                out.append(StepRecord(**json.loads(line)))
    return out


@dataclass
class TraceSummary:
    """analysis.py:165-186."""

    steps: int
    mean_cache_len: float   # mean over steps of the layer-mean length after append
    max_cache_len: int      # max over steps of the layer-max length after append
    eviction_rate: float    # fraction of steps with at least one eviction
    total_evicted: int
    peak_bytes: int
    mean_bytes: float
    confidence_histogram: list[int]  # 20 bins, edges at k/20

    def to_dict(self) -> dict:
        return dict(self.__dict__)


def summarize_trace(records) -> TraceSummary:
    """analysis.py:189-208: deterministic aggregates over one run's step records."""
    if not records:
        raise ValueError("cannot summarize an empty record list")
    step_means = [float(np.mean(r.len_post)) + 1.0 for r in records]
    step_maxes = [max(r.len_post) + 1 for r in records]
    evict_steps = sum(1 for r in records if any(e > 0 for e in r.evicted))
    confs = np.array([r.confidence for r in records])
    hist, _ = np.histogram(confs, bins=20, range=(0.0, 1.0))
    return TraceSummary(
        steps=len(records),
        mean_cache_len=float(np.mean(step_means)),
        max_cache_len=int(max(step_maxes)),
        eviction_rate=evict_steps / len(records),
        total_evicted=int(sum(sum(r.evicted) for r in records)),
        peak_bytes=max(r.memory_bytes for r in records),
        mean_bytes=float(np.mean([r.memory_bytes for r in records])),
        confidence_histogram=[int(x) for x in hist],
    )


def write_snapshot(engine, path, layer: int, seq: int = 0) -> None:
    """CKVS dump of one (layer, sequence) cache of a ConfKVEngine (cache.py:278-301)."""
    c = engine.read_cache(layer, seq)
    write_snapshot_arrays(path, layer, c["keys"], c["values"], c["positions"], c["steps"], c["ema"], c["seen"])


def write_snapshot_arrays(path, layer_id, keys, values, positions, steps, ema, seen) -> None:
    n = int(len(positions))
    heads, dim = (keys.shape[1], keys.shape[2]) if n else (0, 0)
    with open(path, "wb") as f:
        f.write(_SNAP_MAGIC)
        f.write(struct.pack("<4I", int(layer_id), n, heads, dim))
        f.write(np.ascontiguousarray(keys, dtype="<f4").tobytes())
        f.write(np.ascontiguousarray(values, dtype="<f4").tobytes())
        f.write(np.ascontiguousarray(positions, dtype="<i8").tobytes())
        f.write(np.ascontiguousarray(steps, dtype="<i8").tobytes())
        f.write(np.ascontiguousarray(ema, dtype="<f8").tobytes())
        f.write(np.ascontiguousarray(seen, dtype=np.uint8).tobytes())


def read_snapshot(path) -> dict:
    """cache.py:304-326: parse a CKVS snapshot back into arrays."""
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != _SNAP_MAGIC:
            raise ValueError(f"not a cache snapshot (magic {magic!r})")
        layer_id, n, heads, dim = struct.unpack("<4I", f.read(16))
        count = n * heads * dim
        k = np.frombuffer(f.read(4 * count), dtype="<f4").reshape(n, heads, dim)
        v = np.frombuffer(f.read(4 * count), dtype="<f4").reshape(n, heads, dim)
        positions = np.frombuffer(f.read(8 * n), dtype="<i8")
        steps = np.frombuffer(f.read(8 * n), dtype="<i8")
        ema = np.frombuffer(f.read(8 * n), dtype="<f8")
        seen = np.frombuffer(f.read(n), dtype=np.uint8).astype(bool)
    return {"layer_id": layer_id, "valid_len": n, "num_heads": heads, "head_dim": dim, "keys": k, "values": v,
            "positions": positions, "steps": steps, "ema": ema, "seen": seen}


__all__ = ["write_jsonl", "read_jsonl", "TraceSummary", "summarize_trace", "write_snapshot",
           "write_snapshot_arrays", "read_snapshot"]
