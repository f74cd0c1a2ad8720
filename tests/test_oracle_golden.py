"""Pin the CPU oracle to the reference: every fixture under tests/golden was
produced by the unmodified reference (tests/golden/make_golden.py). Equality
here is exact — the oracle reproduces the reference's NumPy ops one for one."""

import json

import numpy as np
import pytest

from oracle import confkv_oracle as O
from oracle import scenarios as S
from paper_2605_24786_b200.config import PolicyConfig


def test_rng_pinned(golden_dir):
    for row in json.load(open(golden_dir / "rng.json")):
        if "seed" in row:
            assert list(O.splitmix_normal(row["seed"], 7)) == row["normal7"]
        else:
            assert O.mix_u64(*row["mix"]) == row["value"]


def test_confidence_pinned(golden_dir):
    rows = json.load(open(golden_dir / "confidence.json"))
    assert len(rows) > 100
    cache = {}
    for r in rows:
        V = r["V"]
        if r["kind"] == "seeded":
            logits = S.step_logits(1000 + V, r["idx"], V)
        else:
            key = ("special", V)
            if key not in cache:
                cache[key] = S.special_logits(V)
            logits = cache[key][r["idx"]]
        assert S.digest(logits) == r["digest"]
        p = O.softmax64(logits, r["temperature"])
        f = O.confidence(p)
        for k in ("entropy_norm", "margin", "margin_sig", "top_prob", "score"):
            assert f[k] == r[k], (r, k, f[k])
        assert O.select_tier(f["score"], 128, 256, 0.7) == r["tier"]
        assert int(np.argmax(p)) == r["argmax"]


@pytest.mark.parametrize("name", list(S.SCENARIOS))
def test_engine_pinned(golden_dir, name):
    meta = json.load(open(golden_dir / f"engine_{name}.json"))
    fx = np.load(golden_dir / f"engine_{name}.npz")
    cfg = PolicyConfig(**S.SCENARIOS[name]["cfg"])
    assert cfg.to_json() == meta["config_json"]
    assert cfg.config_hash() == meta["config_hash"]
    records, outs, kept, eng = S.drive_oracle(name, cfg, O.OracleEngine)

    assert len(records) == len(meta["records"])
    group = S.SCENARIOS[name]["H"] // S.SCENARIOS[name]["Hkv"]
    for mine, ref in zip(records, meta["records"]):
        # the reference (MHA-only) stores K/V expanded to the query heads, so its
        # analytic bytes are `group` x the KV-head bytes
        mine = dict(mine, memory_bytes=mine["memory_bytes"] * group)
        assert mine == ref, (mine["step"], mine, ref)
    assert [S.digest(o) for o in outs] == meta["out_digests"]
    for i, t in enumerate(fx["out_steps"]):
        assert np.array_equal(outs[t], fx["outs"][i])
    assert np.array_equal(np.concatenate(kept), fx["kept_flat"])
    assert [k.shape[0] for k in kept] == list(fx["kept_len"])

    for layer, c in enumerate(eng.caches):
        pre = f"l{layer}_"
        n = int(fx[pre + "n"])
        assert c.n == n
        assert np.array_equal(c.pos[:n], fx[pre + "positions"])
        assert np.array_equal(c.step[:n], fx[pre + "steps"])
        assert np.array_equal(c.ema[:n], fx[pre + "ema"])  # bit-exact EMA
        assert np.array_equal(c.seen[:n], fx[pre + "seen"])
        assert np.array_equal(c.seg[:n], fx[pre + "segment_of"])
        hi = c.seg[:n] == O.HIGH
        assert np.array_equal(c.k[:n][hi], fx[pre + "keys"].astype(np.float32)[hi])
        assert np.array_equal(c.v[:n][hi], fx[pre + "values"].astype(np.float32)[hi])
        assert np.array_equal(c.kc[:n][~hi], fx[pre + "k_codes"][~hi])
        assert np.array_equal(c.vc[:n][~hi], fx[pre + "v_codes"][~hi])
        assert np.array_equal(np.array(c.seg_count, np.int64), fx[pre + "seg_count"])
        if c.seg_count:
            assert np.array_equal(np.stack(c.seg_k), fx[pre + "seg_k_scale"])
            assert np.array_equal(np.stack(c.seg_v), fx[pre + "seg_v_scale"])
