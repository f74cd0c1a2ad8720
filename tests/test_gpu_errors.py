"""Error behaviour at the boundary (reference exception types): argument and
shape errors -> ValueError, config errors -> ConfigError, state misuse / exhausted capacity ->
RuntimeError; and the documented edge behaviour (attention over an empty cache -> zeros)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_24786_b200 import baselines as BL  # noqa: E402
from paper_2605_24786_b200.config import ConfigError, ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402

SHAPE = ModelShape(num_layers=2, num_heads=4, head_dim=32, vocab_size=64, num_kv_heads=2)
CFG = PolicyConfig(n_high=24, n_low=40, protected_p=8, pyramid_n_min=16, fp16_window_w=8)


def _engine(**kw):
    kw.setdefault("batch", 2)
    kw.setdefault("capacity", 48)
    return ConfKVEngine(CFG, SHAPE, quantize=kw.pop("quantize", True), **kw)


def _step(eng, t, q=True):
    B = eng.batch
    kn = torch.randn((2, B, 2, 32)).half().cuda()
    lg = (torch.randn((B, 64)) * 8).cuda()
    qq = torch.randn((2, B, 4, 32)).half().cuda() if q else None
    eng.step(lg, kn, kn, step=t, q=qq)
    return eng.records()


def test_empty_cache_attention_is_zero():
    eng = _engine()
    out = eng.attend(0, torch.randn((2, 4, 32)).half().cuda())
    assert torch.count_nonzero(out) == 0


def test_shape_errors_raise_value_error():
    eng = _engine()
    with pytest.raises(ValueError):
        eng.attend_layers(torch.randn((2, 3, 4, 32)).half().cuda())          # wrong batch
    with pytest.raises(ValueError):
        eng.prefill(torch.randn((2, 2, 5, 3, 32)).half(), torch.randn((2, 2, 5, 3, 32)).half())   # wrong Hkv
    with pytest.raises(ValueError):
        eng.prefill(torch.zeros((2, 2, 60, 2, 32)).half(), torch.zeros((2, 2, 60, 2, 32)).half())  # > capacity
    with pytest.raises(ValueError):
        eng.step(torch.zeros((2, 63)).cuda(), torch.zeros((2, 2, 2, 32)).half(), torch.zeros((2, 2, 2, 32)).half(),
                 step=1)                                                          # short logits
    with pytest.raises(ValueError, match="sum to 1"):
        eng.stage_rows(0, torch.full((2, 4, 1), 0.5, dtype=torch.float64))


def test_config_errors():
    with pytest.raises(ConfigError):
        ConfKVEngine(CFG, SHAPE, batch=1, capacity=30)          # capacity below the budgets
    with pytest.raises(ConfigError):
        ConfKVEngine(CFG, ModelShape(2, 4, 24, 64, num_kv_heads=2), batch=1, capacity=48)   # head_dim 24
    with pytest.raises(ValueError):
        BL.SlidingWindowPolicy(CFG, SHAPE, window=0)
    with pytest.raises(ValueError):
        BL.HeavyHitterPolicy(CFG, SHAPE, cap=4)                 # cap below the protected window
    with pytest.raises(ValueError, match="mode"):
        BL.MatchedRatePolicy(CFG, SHAPE, [], "bogus")


def test_capacity_exhaustion_raises_runtime_error():
    # the full-cache baseline never evicts: the 49th entry overflows a 48-entry capacity
    eng = BL.FullCachePolicy(CFG, SHAPE, batch=1, capacity=48)
    eng.begin_prefill(40)
    z = torch.randn((2, 1, 40, 2, 32)).half()
    eng.prefill(z, z)
    for t in range(1, 9):
        _step(eng, t)
    with pytest.raises(RuntimeError, match="capacity"):
        _step(eng, 9)


def test_single_entry_segments_need_no_pool():
    # every step demotes one entry into a new single-entry segment: those take no lossy-pool
    # (scale-row) slot, so a pool of 1 (the prefill's bulk segment) suffices
    eng = _engine(batch=1, max_segments=1)
    eng.begin_prefill(20)
    z = torch.randn((2, 1, 20, 2, 32)).half()
    eng.prefill(z, z)
    for t in range(1, 30):
        _step(eng, t)
    assert eng.records()[0].int8[0] > 0


def test_matched_schedule_overdraw_raises_value_error():
    eng = BL.MatchedRatePolicy(CFG, SHAPE, [(1, 0, 100)], "recency_only", batch=1, capacity=48)
    eng.begin_prefill(20)
    z = torch.randn((2, 1, 20, 2, 32)).half()
    eng.prefill(z, z)
    with pytest.raises(ValueError, match="schedule"):
        _step(eng, 1)


def test_reset_empties_every_cache():
    eng = _engine()
    eng.begin_prefill(30)
    z = torch.randn((2, 2, 30, 2, 32)).half()
    eng.prefill(z, z)
    _step(eng, 1)
    eng.reset()
    for layer in range(2):
        for b in range(2):
            assert eng.read_cache(layer, b)["valid_len"] == 0
    eng.begin_prefill(5)
    eng.prefill(z[:, :, :5].contiguous(), z[:, :, :5].contiguous())
    recs = _step(eng, 1)
    assert recs[0].len_pre == [5, 5] and recs[0].step == 1
    assert np.all([r.len_post[0] == 5 for r in recs])
