"""Drop-in at the reference's own driver boundary: `run_decode` + `TraceDriver`
(simulator.py:408-478) driving a policy through `policy.caches[l].valid_len / .positions`
and `policy.step(logits, attention_rows, new_kv, t) -> StepRecord` (policy.py:187-224).

Fixtures (tests/golden/rundecode_*) were written by the UNMODIFIED reference
(`make_golden.py --run-decode`): retention_suite needle traces and the StepRecord JSONL
`run_decode` produced for confkv / confkv-int8 / confkv-l.
- CPU: the test-side restatement of the protocol (tests/trace_protocol.py) driving the
  oracle reproduces the reference's JSONL exactly (pins the restatement).
- GPU: the same loop drives `ConfKVEngine` (batch 1) unchanged -- the records must equal the
  reference's (integers exactly, fp64 confidence features to 1e-12) and the needle verdict too.
"""

from __future__ import annotations

import io
import json

import numpy as np
import pytest

from oracle import confkv_oracle as O
from paper_2605_24786_b200.config import ModelShape, PolicyConfig
from tests.trace_protocol import Trace, TraceDriver, compare_jsonl, run_decode


def _runs(golden_dir):
    meta = json.loads((golden_dir / "rundecode.json").read_text())
    return meta["runs"]


class _Rec(dict):
    @property
    def token(self):
        return self["token"]

    def to_dict(self):
        return dict(self)


class _OracleCacheView:
    def __init__(self, cache):
        self._c = cache

    @property
    def valid_len(self):
        return self._c.n

    @property
    def positions(self):
        return self._c.pos[: self._c.n]


class OraclePolicy:
    """The oracle behind the reference's DecodePolicy surface (CPU pin of the protocol)."""

    def __init__(self, cfg, trace: Trace, quantize: bool):
        self.e = O.OracleEngine(cfg, trace.num_layers, trace.num_heads, trace.head_dim, trace.vocab_size,
                                quantize=quantize)
        self.caches = [_OracleCacheView(c) for c in self.e.caches]

    def begin_prefill(self, n):
        self.e.begin_prefill(n)

    def append_prefill(self, layer, k, v, pos):
        self.e.append_prefill(layer, k, v, pos)

    def step(self, logits, rows, new_kv, t):
        return _Rec(self.e.step(logits, rows, new_kv, t))


@pytest.mark.parametrize("run", range(6))
def test_protocol_restatement_reproduces_reference_jsonl(golden_dir, run):
    r = _runs(golden_dir)[run]
    trace = Trace(golden_dir / f"rundecode_trace{r['trace']}.jsonl")
    cfg = PolicyConfig(pyramid_enabled=r["policy"] == "confkv-l")
    pol = OraclePolicy(cfg, trace, quantize=r["policy"] != "confkv")
    sink = io.StringIO()
    _, retained = run_decode(pol, TraceDriver(trace), r["steps"], sink=sink)
    ref = (golden_dir / r["jsonl"]).read_text().splitlines()
    compare_jsonl(sink.getvalue().splitlines(), ref, rtol=0.0, what=f"oracle {r['policy']}")
    assert retained == r["needle_retained"]


@pytest.mark.gpu
@pytest.mark.parametrize("run", range(6))
def test_engine_is_a_drop_in_for_run_decode(golden_dir, run):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2605_24786_b200.engine import ConfKVEngine, StepRecord
    r = _runs(golden_dir)[run]
    trace = Trace(golden_dir / f"rundecode_trace{r['trace']}.jsonl")
    cfg = PolicyConfig(pyramid_enabled=r["policy"] == "confkv-l")
    shape = ModelShape(trace.num_layers, trace.num_heads, trace.head_dim, trace.vocab_size)
    # constructed the way cli.py:82-88 constructs the reference's policies
    eng = ConfKVEngine(cfg, shape, quantize=r["policy"] != "confkv")
    assert eng.name == r["policy"]
    sink = io.StringIO()
    recs, retained = run_decode(eng, TraceDriver(trace), r["steps"], sink=sink)
    assert all(isinstance(x, StepRecord) for x in recs)
    ref = (golden_dir / r["jsonl"]).read_text().splitlines()
    compare_jsonl(sink.getvalue().splitlines(), ref, rtol=1e-12, what=f"engine {r['policy']}")
    assert retained == r["needle_retained"]
    # the facade's host views agree with the device state
    for layer, c in enumerate(eng.caches):
        st = eng.read_cache(layer, 0)
        assert c.valid_len == st["valid_len"]
        assert np.array_equal(c.positions, st["positions"])
    eng.close()
