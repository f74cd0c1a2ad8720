"""F4: the oracle's comparison policies (OracleBaseline, restating baselines.py) pinned to
fixtures written by the unmodified reference (make_golden.py --baselines)."""

import json

import numpy as np
import pytest

from oracle import confkv_oracle as O
from oracle import scenarios as S
from paper_2605_24786_b200.config import PolicyConfig

TAGS = ["full", "sliding", "heavy_hitter", "matched_random", "matched_recency_only", "matched_attention_only"]


def drive_baseline(meta, capacity=64):
    spec = S.SCENARIOS[meta["scenario"]]
    L, H, Hkv, D, V, seed = spec["L"], spec["H"], spec["Hkv"], spec["D"], spec["V"], spec["seed"]
    cfg = PolicyConfig(**spec["cfg"])
    kw = dict(meta["kwargs"])
    if meta["kind"] == "matched":
        kw["schedule"] = [tuple(e) for e in meta["schedule"]]
    eng = O.OracleBaseline(cfg, L, H, D, V, meta["kind"], kv_heads=Hkv, capacity=capacity, **kw)
    eng.begin_prefill(spec["prefill"])
    for layer in range(L):
        k, v = S.scenario_prefill_kv(spec, seed, layer)
        for pos in range(spec["prefill"]):
            eng.append_prefill(layer, k[pos], v[pos], pos)
    recs, kept = [], []
    for t in range(1, spec["steps"] + 1):
        rows = [eng.attend(layer, S.scenario_q(spec, seed, t, layer))[1] for layer in range(L)]
        new_kv = [S.step_kv(seed, t, layer, Hkv, D) for layer in range(L)]
        rec, kp = eng.step(S.step_logits(seed, t, V), rows, new_kv, t, return_kept=True)
        recs.append(rec)
        kept.extend(kp)
    return recs, kept, eng


@pytest.mark.parametrize("tag", TAGS)
def test_baseline_pinned(golden_dir, tag):
    meta = json.load(open(golden_dir / f"baseline_{tag}.json"))
    fx = np.load(golden_dir / f"baseline_{tag}.npz")
    recs, kept, eng = drive_baseline(meta)
    group = S.SCENARIOS[meta["scenario"]]["H"] // S.SCENARIOS[meta["scenario"]]["Hkv"]
    for mine, ref in zip(recs, meta["records"]):
        assert dict(mine, memory_bytes=mine["memory_bytes"] * group) == ref, mine["step"]
    assert np.array_equal(np.concatenate(kept), fx["kept_flat"])
    for layer, c in enumerate(eng.caches):
        n = c.n
        pre = f"l{layer}_"
        assert np.array_equal(c.pos[:n], fx[pre + "positions"])
        assert np.array_equal(c.step[:n], fx[pre + "steps"])
        assert np.array_equal(c.ema[:n], fx[pre + "ema"])
        assert np.array_equal(c.seen[:n], fx[pre + "seen"])
        assert np.array_equal(c.cum[:n], fx[pre + "cum"])


def test_baseline_errors():
    cfg = PolicyConfig()
    with pytest.raises(ValueError, match="mode"):
        O.OracleBaseline(cfg, 1, 1, 16, 8, "matched", schedule=[], mode="bogus")
    with pytest.raises(ValueError, match="duplicate"):
        O.OracleBaseline(cfg, 1, 1, 16, 8, "matched", schedule=[(1, 0, 1), (1, 0, 2)], mode="random")
    c = O.OracleCache(1, 4)
    with pytest.raises(ValueError, match="window"):
        O.sliding_window_step(c, 0)
    with pytest.raises(ValueError, match="cap"):
        O.heavy_hitter_step(c, 3, 4)
