"""F4 on the GPU: the comparison policies (full, sliding window, heavy hitter, matched-rate
random / recency / attention) on the same K2/K3 kernels, (1) bit-exact against the oracle
fed the GPU's attention weights, and (2) with the reference's attention rows (trace-driver
path), against the fixtures the unmodified reference wrote (make_golden.py --baselines)."""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import confkv_oracle as O  # noqa: E402
from oracle import scenarios as S  # noqa: E402
from paper_2605_24786_b200 import baselines as BL  # noqa: E402
from tests.gpu_driver import run_scenario  # noqa: E402

TAGS = ["full", "sliding", "heavy_hitter", "matched_random", "matched_recency_only", "matched_attention_only"]


def _factories(meta):
    spec = S.SCENARIOS[meta["scenario"]]
    L, H, Hkv, D, V = spec["L"], spec["H"], spec["Hkv"], spec["D"], spec["V"]
    kind, kw = meta["kind"], dict(meta["kwargs"])
    full_cap = spec["prefill"] + spec["steps"] + 2

    def make_engine(cfg, shape, batch, cap):
        if kind == "full":
            return BL.FullCachePolicy(cfg, shape, batch=batch, capacity=full_cap)
        if kind == "sliding":
            return BL.SlidingWindowPolicy(cfg, shape, kw["window"], batch=batch, capacity=cap)
        if kind == "heavy_hitter":
            return BL.HeavyHitterPolicy(cfg, shape, kw["cap"], batch=batch, capacity=cap)
        return BL.MatchedRatePolicy(cfg, shape, [tuple(e) for e in meta["schedule"]], kw["mode"], batch=batch,
                                    capacity=cap)

    def make_oracle(cfg):
        okw = dict(kw)
        if kind == "matched":
            okw["schedule"] = [tuple(e) for e in meta["schedule"]]
        return O.OracleBaseline(cfg, L, H, D, V, kind, kv_heads=Hkv, **okw)

    return make_engine, make_oracle


@pytest.mark.parametrize("tag", TAGS)
def test_baseline_vs_oracle(golden_dir, tag):
    meta = json.load(open(golden_dir / f"baseline_{tag}.json"))
    me, mo = _factories(meta)
    r = run_scenario(meta["scenario"], batch=2, make_engine=me, make_oracle=mo, check_every=40)
    assert r["worst_attn_rel"] < 1e-3


@pytest.mark.parametrize("tag", TAGS)
def test_baseline_vs_reference_fixture(golden_dir, tag):
    meta = json.load(open(golden_dir / f"baseline_{tag}.json"))
    fx = np.load(golden_dir / f"baseline_{tag}.npz")
    me, mo = _factories(meta)
    spec = S.SCENARIOS[meta["scenario"]]
    group = spec["H"] // spec["Hkv"]

    def on_step(t, recs):
        g, ref = recs[0].to_dict(), meta["records"][t - 1]
        for k in ("step", "budget", "len_pre", "len_post", "evicted", "int8", "token"):
            assert g[k] == ref[k], (t, k, g[k], ref[k])
        assert g["memory_bytes"] * group == ref["memory_bytes"], t

    def on_end(eng):
        for layer in range(spec["L"]):
            c = eng.read_cache(layer, 0)
            pre = f"l{layer}_"
            assert np.array_equal(c["positions"], fx[pre + "positions"])
            assert np.array_equal(c["steps"], fx[pre + "steps"])
            assert np.array_equal(c["ema"], fx[pre + "ema"])
            assert np.array_equal(c["seen"], fx[pre + "seen"])
            if "cum" in c:
                assert np.array_equal(c["cum"], fx[pre + "cum"])

    run_scenario(meta["scenario"], batch=1, use_gpu_rows=False, make_engine=me, make_oracle=mo,
                 on_step=on_step, on_end=on_end, check_every=80)


def test_schedule_recording_roundtrip(tmp_path):
    """ConfKVEngine(record_schedule=True) records the per-(step, layer) eviction counts the
    matched-rate replay consumes; write_schedule / read_schedule round-trip them."""
    from paper_2605_24786_b200.config import ModelShape, PolicyConfig
    from paper_2605_24786_b200.engine import ConfKVEngine
    cfg = PolicyConfig(n_high=24, n_low=40, protected_p=8, pyramid_n_min=16)
    shape = ModelShape(2, 2, 16, 50)
    eng = ConfKVEngine(cfg, shape, record_schedule=True, batch=1, capacity=64)
    eng.begin_prefill(40)
    z = torch.randn((2, 1, 40, 2, 16)).half()
    eng.prefill(z, z)
    total = 0
    for t in range(1, 30):
        q = torch.randn((2, 1, 2, 16)).half().cuda()
        kn = torch.randn((2, 1, 2, 16)).half()
        eng.step((torch.randn((1, 50)) * (8 if t % 3 else 0.5)), kn, kn, step=t, q=q)
        total += sum(eng.records()[0].evicted)
    assert sum(e.evict_count for e in eng.schedule) == total > 0
    BL.write_schedule(eng.schedule, tmp_path / "s.jsonl")
    assert BL.read_schedule(tmp_path / "s.jsonl") == eng.schedule
