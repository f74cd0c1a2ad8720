"""Host config parity with the reference config.py (SPEC:46-48 examples + JSON/hash)."""

import json

import pytest

from paper_2605_24786_b200.config import (ConfigError, ModelShape, PolicyConfig, budget_table, load_config,
                                          preset, pyramid_budget)


def test_defaults_spec_46():
    c = load_config("{}")
    assert (c.tau, c.n_high, c.n_low, c.protected_p, c.alpha, c.ema_lambda, c.fp16_window_w,
            c.block_size_b, c.confidence_weights, c.pyramid_beta, c.pyramid_n_min) == (
        0.7, 128, 256, 32, 0.65, 0.90, 128, 128, (0.4, 0.3, 0.3), 0.5, 96)


@pytest.mark.parametrize("doc,frag", [
    ('{"n_high":512,"n_low":256}', "n_high <= n_low"),
    ('{"w_entropy":0.5,"w_margin":0.5,"w_top":0.5}', "sum to 1"),
    ('{"bogus": 1}', "unknown config keys"),
    ('{"n_high": 1.5}', "must be an integer"),
    ('{"n_high": true}', "must be an integer"),
    ('[1]', "JSON object"),
    ('{', "not valid JSON"),
    ('{"protected_p": 200}', "protected_p <= pyramid_n_min"),
    ('{"tau": 1.5}', "tau must lie"),
    ('{"sampling_mode": {"temperature": 0.0}}', "temperature"),
    ('{"sampling_mode": "nucleus"}', "unknown sampling_mode"),
])
def test_rejections(doc, frag):
    with pytest.raises(ConfigError, match=frag.replace("(", r"\(")):
        load_config(doc)


def test_roundtrip_and_hash_stable():
    c = preset("niah")
    d = json.loads(c.to_json())
    c2 = load_config(json.dumps(d))
    assert c2 == c and c2.config_hash() == c.config_hash()
    t = load_config('{"sampling_mode": {"temperature": 0.7}}')
    assert t.sampling_mode == "temperature" and t.temperature == 0.7
    assert load_config(t.to_json()) == t


def test_reference_hash_matches_when_available():
    ref = pytest.importorskip("confkv.config") if False else None  # reference is only in the build container
    import os
    import sys
    path = "/root/reference/pkg/src"
    if not os.path.isdir(path):
        pytest.skip("reference not mounted")
    sys.path.insert(0, path)
    from confkv import config as R
    for name in ("wikitext", "niah", "vwa"):
        assert R.preset(name).to_json() == preset(name).to_json()
        assert R.preset(name).config_hash() == preset(name).config_hash()
    for doc in ('{"n_high": 100, "pyramid_enabled": true}', '{"sampling_mode": {"temperature": 1.3}}'):
        assert R.load_config(doc).to_json() == load_config(doc).to_json()


def test_pyramid_spec_364():
    shape = ModelShape(num_layers=12)
    assert pyramid_budget(0, shape, 128, 0.5, 96) == 128
    assert pyramid_budget(4, shape, 128, 0.5, 96) == 101
    assert pyramid_budget(12, shape, 128, 0.5, 96) == 96
    vals = [pyramid_budget(l, shape, 128, 0.5, 96) for l in range(13)]
    assert vals == sorted(vals, reverse=True)
    with pytest.raises(ValueError):
        pyramid_budget(13, shape, 128, 0.5, 96)


def test_budget_table():
    cfg = PolicyConfig(pyramid_enabled=True)
    tab = budget_table(cfg, ModelShape(num_layers=12))
    assert tab[0] == (128, 256) and tab[4] == (101, 203)
    assert budget_table(PolicyConfig(), ModelShape(num_layers=3)) == [(128, 256)] * 3


def test_shape_gqa():
    s = ModelShape(num_layers=32, num_heads=32, head_dim=128, vocab_size=128256, num_kv_heads=8)
    assert s.kv_heads == 8 and s.group == 4
    with pytest.raises(ConfigError):
        ModelShape(num_heads=6, num_kv_heads=4)
    with pytest.raises(ConfigError):
        ModelShape(num_layers=0)
