"""Host-side StepRecord parsing (engine._parse_records): the NumPy-vectorised path used for
>= 96 (layer, sequence) records must produce exactly what the per-record ctypes loop produces
(values, memory_bytes, schedules, and which status raises), on CPU with synthetic records."""

import random

import pytest

from paper_2605_24786_b200 import _lib
from paper_2605_24786_b200.baselines import SlidingWindowPolicy
from paper_2605_24786_b200.config import ModelShape, PolicyConfig
from paper_2605_24786_b200.engine import ConfKVEngine


def _host_engine(cls, L, B, schedules):
    eng = cls.__new__(cls)          # host-only: no device state is touched by the parser
    eng.shape = ModelShape(L, 8, 128, 1000, num_kv_heads=4)
    eng.batch = B
    eng.config = PolicyConfig()
    eng.schedules = [[] for _ in range(B)] if schedules else None
    if cls is SlidingWindowPolicy:
        eng.window = 300
    return eng


def _records(L, B, rng, status=None):
    rl = (_lib.CkvLayerRecord * (L * B))()
    rs = (_lib.CkvSeqRecord * B)()
    for r in rl:
        r.len_pre = rng.randint(0, 5000)
        r.len_post = rng.randint(0, 5000)
        r.evicted = rng.choice([0, 0, 1, 3])
        r.int8_count = rng.randint(0, 4000)
        r.len_after = r.int8_count + rng.randint(0, 300)
        r.num_segments = rng.randint(0, 4000)
    for q in rs:
        q.score, q.entropy_norm, q.margin = rng.random(), rng.random(), rng.random() * 9
        q.margin_sig, q.top_prob = rng.random(), rng.random()
        q.tier_high, q.token = rng.randint(0, 1), rng.randint(0, 999)
    if status is not None:
        b, layer, bits = status
        if layer is None:
            rs[b].status = bits
        else:
            rl[layer * B + b].status = bits
    return rl, rs


@pytest.mark.parametrize("L,B", [(32, 8), (4, 30), (64, 2)])
@pytest.mark.parametrize("cls", [ConfKVEngine, SlidingWindowPolicy])
@pytest.mark.parametrize("schedules", [False, True])
def test_vectorised_parse_matches_loop(L, B, cls, schedules):
    assert L * B >= 96                        # the vectorised path
    rng = random.Random(L * 1000 + B)
    rl, rs = _records(L, B, rng)
    a = _host_engine(cls, L, B, schedules)
    b = _host_engine(cls, L, B, schedules)
    ra = a._parse_records(rl, rs, 7)
    rb = b._parse_records_loop(rl, rs, 7)
    assert ra == rb
    assert a.schedules == b.schedules


@pytest.mark.parametrize("bits,exc", [(_lib.ST_NONFINITE, ValueError), (_lib.ST_NOATTEND, RuntimeError),
                                      (_lib.ST_SCHEDULE, ValueError), (_lib.ST_OVERFLOW, RuntimeError),
                                      (_lib.ST_SEGOVERFLOW, RuntimeError)])
@pytest.mark.parametrize("where", [(3, 5), (6, None)])
def test_vectorised_parse_raises_like_loop(bits, exc, where):
    L, B = 16, 8
    rl, rs = _records(L, B, random.Random(5), status=(where[0], where[1], bits))
    for parse in ("_parse_records", "_parse_records_loop"):
        eng = _host_engine(ConfKVEngine, L, B, False)
        with pytest.raises(exc):
            getattr(eng, parse)(rl, rs, 1)


def test_kept_maps_compact_form():
    """HostPipeline.kept() returns KeptMaps: victim lists + pre-step lengths; indexing
    materialises each cache's kept map as the complement of its victims (policy.py:117-127)."""
    import numpy as np

    from paper_2605_24786_b200.engine import KeptMaps, kept_from_victims
    rng = np.random.default_rng(3)
    L, B, vmax = 3, 2, 4
    len_pre = rng.integers(10, 50, size=(L, B)).astype(np.int32)
    ev = rng.integers(0, vmax + 1, size=(L, B)).astype(np.int32)
    ev[1, 1] = 7                                   # one cache beyond the D2H head
    head = np.zeros((L, B, vmax), np.int32)
    over, full = {}, {}
    for layer in range(L):
        for b in range(B):
            v = np.sort(rng.choice(len_pre[layer, b], ev[layer, b], replace=False)).astype(np.int32)
            full[(layer, b)] = v
            if ev[layer, b] > vmax:
                over[(layer, b)] = v
            else:
                head[layer, b, :ev[layer, b]] = v
    km = KeptMaps(len_pre, ev, head, over)
    assert len(km) == L
    for layer, row in enumerate(km):
        for b in range(B):
            exp = np.setdiff1d(np.arange(len_pre[layer, b]), full[(layer, b)]).astype(np.int32)
            assert np.array_equal(row[b], exp)
            assert np.array_equal(km.victims(layer, b), full[(layer, b)])
            assert np.array_equal(kept_from_victims(len_pre[layer, b], full[(layer, b)]), exp)
