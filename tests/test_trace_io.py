"""F3: StepRecord JSONL, TraceSummary and CKVS snapshots against fixtures written by the
unmodified reference (tests/golden/make_golden.py: trace_*.jsonl, summary_*.json,
snap_*.ckvs)."""

import io
import json

import numpy as np
import pytest

from oracle import confkv_oracle as O
from oracle import scenarios as S
from paper_2605_24786_b200.config import PolicyConfig
from paper_2605_24786_b200.trace import (read_jsonl, read_snapshot, summarize_trace, write_jsonl,
                                         write_snapshot_arrays)

IO = ["int8_mha", "fp16_mha"]


@pytest.mark.parametrize("name", IO)
def test_jsonl_roundtrip_and_summary(golden_dir, name):
    path = golden_dir / f"trace_{name}.jsonl"
    recs = read_jsonl(path)
    assert len(recs) == S.SCENARIOS[name]["steps"]
    buf = io.StringIO()
    write_jsonl(recs, buf)
    assert buf.getvalue() == path.read_text()           # byte-identical schema and key order
    ref = json.load(open(golden_dir / f"summary_{name}.json"))
    assert summarize_trace(recs).to_dict() == ref         # exact aggregates
    with pytest.raises(ValueError):
        summarize_trace([])


@pytest.mark.parametrize("name", IO)
def test_snapshot_roundtrip_matches_oracle(golden_dir, name, tmp_path):
    spec = S.SCENARIOS[name]
    cfg = PolicyConfig(**spec["cfg"])
    _, _, _, eng = S.drive_oracle(name, cfg, O.OracleEngine)
    for layer in range(spec["L"]):
        path = golden_dir / f"snap_{name}_l{layer}.ckvs"
        snap = read_snapshot(path)
        c = eng.caches[layer]
        n = c.n
        assert snap["layer_id"] == layer and snap["valid_len"] == n
        assert (snap["num_heads"], snap["head_dim"]) == (spec["Hkv"], spec["D"])
        kd, vd = c.dequant_kv(0, n)
        assert np.array_equal(snap["keys"], kd) and np.array_equal(snap["values"], vd)
        assert np.array_equal(snap["positions"], c.pos[:n]) and np.array_equal(snap["steps"], c.step[:n])
        assert np.array_equal(snap["ema"], c.ema[:n]) and np.array_equal(snap["seen"], c.seen[:n])
        out = tmp_path / "x.ckvs"
        write_snapshot_arrays(out, layer, snap["keys"], snap["values"], snap["positions"], snap["steps"],
                              snap["ema"], snap["seen"])
        assert out.read_bytes() == path.read_bytes()


def test_snapshot_bad_magic(tmp_path):
    p = tmp_path / "bad.ckvs"
    p.write_bytes(b"NOPE" + bytes(16))
    with pytest.raises(ValueError, match="snapshot"):
        read_snapshot(p)
