"""The reference's decode-driver protocol, restated for the tests (TEST INFRASTRUCTURE).

`run_decode` (simulator.py:448-478), `TraceDriver` (simulator.py:408-437) and the parts of
`SyntheticTrace` it uses (`read_jsonl` :173-208, `kv_draw` :128-132, `attention_rows`
:134-146). The GPU box has no `/root/reference`, so the drop-in test drives the B200 engine
through this restatement over trace files the reference wrote (tests/golden/rundecode_*),
and a CPU test pins the restatement by driving the oracle through it against the
reference's own output JSONL.

A policy here is anything with the reference's `DecodePolicy` surface: `begin_prefill(n)`,
`append_prefill(layer, k, v, pos)`, `caches[l].valid_len` / `.positions`,
`step(logits, attention_rows, new_kv, step) -> record` with `record.token` and
`record.to_dict()`.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from oracle.confkv_oracle import mix_u64, splitmix_normal


@dataclass
class TraceStep:
    logits: np.ndarray
    spike: bool


class Trace:
    """SyntheticTrace.read_jsonl (simulator.py:173-208) + kv_draw / attention_rows."""

    def __init__(self, path):
        with open(path) as f:
            header = json.loads(f.readline())
            if header.get("kind") != "confkv-trace":
                raise ValueError(f"{path} is not a trace file")
            self.steps = []
            for line in f:
                if line.strip():
                    d = json.loads(line)
                    self.steps.append(TraceStep(np.asarray(d["logits"], dtype=np.float64), bool(d["spike"])))
        self.num_layers, self.num_heads = header["num_layers"], header["num_heads"]
        self.head_dim, self.vocab_size = header["head_dim"], header["vocab_size"]
        self.prefill_len = header["prefill_len"]
        self.needle_position, self.query_step = header.get("needle_position"), header.get("query_step")
        self.spike_mass = header.get("spike_mass", 0.0)
        self.kv_seed = header["kv_seed"]

    def __len__(self):
        return len(self.steps)

    def kv_draw(self, phase: int, index: int, layer: int):
        """simulator.py:128-132: SeededRng(mix_u64(kv_seed, phase, index, layer)).normal."""
        h, hd = self.num_heads, self.head_dim
        buf = splitmix_normal(mix_u64(self.kv_seed, phase, index, layer), 2 * h * hd).reshape(2, h, hd)
        return buf[0].astype(np.float32), buf[1].astype(np.float32)

    def attention_rows(self, step: int, cache) -> np.ndarray:
        """simulator.py:134-146."""
        n = cache.valid_len
        row = np.full(n, 1.0 / n)
        ts = self.steps[step - 1]
        if ts.spike and self.needle_position is not None:
            hits = np.nonzero(cache.positions[:n] == self.needle_position)[0]
            if hits.size == 1 and n > 1:
                row = np.full(n, (1.0 - self.spike_mass) / (n - 1))
                row[hits[0]] = self.spike_mass
            elif hits.size == 1:
                row = np.array([1.0])
        return np.broadcast_to(row, (self.num_heads, n)).copy()


class TraceDriver:
    """simulator.py:408-437."""

    def __init__(self, trace: Trace):
        self.trace = trace
        self.prefill_len = trace.prefill_len
        self.needle_position, self.query_step = trace.needle_position, trace.query_step

    def prefill(self, policy) -> None:
        for pos in range(self.trace.prefill_len):
            for layer in range(self.trace.num_layers):
                k, v = self.trace.kv_draw(0, pos, layer)
                policy.append_prefill(layer, k, v, pos)

    def first_token(self) -> int:
        return 0

    def step_inputs(self, step: int, caches, token: int):
        if step > len(self.trace.steps):
            raise RuntimeError(f"trace exhausted: step {step} > {len(self.trace.steps)} scripted steps")
        ts = self.trace.steps[step - 1]
        rows = [self.trace.attention_rows(step, c) for c in caches]
        new_kv = [self.trace.kv_draw(1, step, layer) for layer in range(self.trace.num_layers)]
        return ts.logits, rows, new_kv


def run_decode(policy, driver, steps: int, sink=None):
    """simulator.py:448-478. Returns (records, needle_retained)."""
    policy.begin_prefill(driver.prefill_len)
    driver.prefill(policy)
    token = driver.first_token()
    records, retained = [], None
    for t in range(1, steps + 1):
        logits, rows, new_kv = driver.step_inputs(t, policy.caches, token)
        if driver.query_step == t and driver.needle_position is not None:
            retained = all((c.positions[: c.valid_len] == driver.needle_position).any() for c in policy.caches)
        rec = policy.step(logits, rows, new_kv, t)
        records.append(rec)
        if sink is not None:
            sink.write(json.dumps(rec.to_dict()) + "\n")
        token = rec.token
    return records, retained


INT_FIELDS = ("step", "budget", "len_pre", "len_post", "evicted", "int8", "memory_bytes", "token")
FLOAT_FIELDS = ("confidence", "entropy_norm", "margin", "margin_sig", "top_prob")


def compare_jsonl(got_lines, ref_lines, rtol: float = 1e-12, what: str = ""):
    """StepRecord JSONL rows: integer fields exactly, float fields within rtol."""
    assert len(got_lines) == len(ref_lines), f"{what}: {len(got_lines)} rows vs {len(ref_lines)}"
    for i, (g, r) in enumerate(zip(got_lines, ref_lines)):
        g, r = json.loads(g), json.loads(r)
        assert list(g) == list(r), f"{what} row {i}: keys {list(g)} vs {list(r)}"
        for k in INT_FIELDS:
            assert g[k] == r[k], f"{what} step {r['step']} {k}: {g[k]} != {r[k]}"
        for k in FLOAT_FIELDS:
            assert abs(g[k] - r[k]) <= rtol * max(1.0, abs(r[k])), f"{what} step {r['step']} {k}: {g[k]} vs {r[k]}"
