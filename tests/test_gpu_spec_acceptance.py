"""The reference SPEC's acceptance checks on the GPU path:

- SPEC:651 eviction fuzz -- 10,240 random caches (n, N, P, alpha) through K3 (rows staged with
  ckv_stage_rows, tie-heavy masses so composite ties are frequent) against an independent full
  sort of (composite, index): lowest index first on ties (policy.py:103-114).
- SPEC:650 tiled attention == naive attention -- 1,000+ random (D, group, n, INT8) cases: K2's
  outputs and weights against a naive fp64 softmax(q k^T / sqrt(d)) v over the same
  (dequantised) cache (attention.py:33-57), within the north star's 1e-3 (fp32 accumulation).
- SPEC:653 INT8 round trip -- over 10^6 demoted elements |x - code*scale| <= scale/2, codes and
  scales bit-exact with quantize_segment (quantizer.py:16-34).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import confkv_oracle as O  # noqa: E402
from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402


def _tie_rows(rng, B, H, n):
    """Attention rows [B, H, n] whose head mean takes few distinct values: every head of a
    sequence gets the same row w/sum(w) with w in {1, 2, 3} (or all-equal rows)."""
    rows = np.empty((B, H, n))
    for b in range(B):
        levels = int(rng.integers(1, 4))
        w = rng.integers(1, levels + 1, size=n).astype(np.float64)
        rows[b] = (w / w.sum())[None, :]
    return rows


def _expected_kept(ema, steps, n, N, P, alpha):
    """Independent full sort (not np.lexsort): victims = the n - N smallest
    (composite, index) pairs among the first n - P entries."""
    cut = n - P
    comp = O.composite(ema[:cut], steps[:cut], alpha)
    order = sorted(range(cut), key=lambda i: (comp[i], i))
    vict = set(order[: n - N])
    return np.array([i for i in range(n) if i not in vict], np.int32)


@pytest.mark.parametrize("k3t", ["0", "256"], ids=["k3_auto", "k3_256"])
def test_eviction_fuzz_10k(k3t, monkeypatch):
    """K3 at its default block size and forced to 256-thread CTAs (the many-short-caches launch)."""
    monkeypatch.setenv("CKV_K3T", k3t)
    rng = np.random.default_rng(651)
    L, B, H, D, V = 4, 64, 4, 16, 64
    cases = ties = 0
    for it in range(40):
        N = int(rng.integers(4, 700))
        P = int(rng.integers(0, N + 1))
        n = N + (1 if it % 5 == 0 else int(rng.integers(1, 500)))   # excess 1: the arg-min path
        alpha = [0.0, 1.0, 0.5, 0.65, float(rng.random())][it % 5]
        cfg = PolicyConfig(n_high=N, n_low=N, protected_p=P, pyramid_n_min=P, alpha=alpha)
        eng = ConfKVEngine(cfg, ModelShape(L, H, D, V), quantize=False, batch=B, capacity=n + 2)
        eng.begin_prefill(n)
        z = torch.zeros((L, B, n, H, D), dtype=torch.half)
        eng.prefill(z, z)
        rows = [_tie_rows(rng, B, H, n) for _ in range(L)]
        for layer in range(L):
            eng.stage_rows(layer, rows[layer])
        zk = torch.zeros((L, B, H, D), dtype=torch.half)
        res = eng.step(torch.zeros((B, V)), zk, zk, step=1)
        eng.records()
        km, kl = res.kept_map.cpu().numpy(), res.kept_len.cpu().numpy()
        steps = np.arange(n, dtype=np.int64) - n
        for layer in range(L):
            for b in range(B):
                ema = rows[layer][b].mean(axis=0)   # cold start: ema = head mean (cache.py:175)
                exp = _expected_kept(ema, steps, n, N, P, alpha)
                got = km[layer, b, : kl[layer, b]]
                assert np.array_equal(got, exp), (it, layer, b, n, N, P, alpha)
                comp = O.composite(ema[: n - P], steps[: n - P], alpha)
                ties += int(comp.size - np.unique(comp).size)
                cases += 1
        eng.close()
    assert cases >= 10000
    assert ties > 100000   # composite ties were exercised heavily


def _naive(q, k, v, group):
    """attention.py:33-57 (naive softmax, fp64) with KV heads repeated over the group."""
    k = np.repeat(k.astype(np.float64), group, axis=1)
    v = np.repeat(v.astype(np.float64), group, axis=1)
    s = np.einsum("hd,nhd->hn", q.astype(np.float64), k) / np.sqrt(q.shape[1])
    e = np.exp(s - s.max(axis=1, keepdims=True))
    w = e / e.sum(axis=1, keepdims=True)
    return np.einsum("hn,nhd->hd", w, v), w


@pytest.mark.parametrize("quantize", [False, True], ids=["fp16", "int8"])
def test_tiled_equals_naive_1000(quantize):
    rng = np.random.default_rng(650 + quantize)
    L, B = 2, 26
    cases = 0
    worst_o = worst_w = 0.0
    for it in range(20):
        D = [16, 32, 64, 128][it % 4]
        G = [1, 2, 4, 5, 8][(it // 4) % 5]
        Hkv = 2 if G > 2 else 3
        H = Hkv * G
        n = int(rng.integers(1, 1800))
        W = int(rng.integers(0, n + 1)) if quantize else 128
        cfg = PolicyConfig(n_high=n + 8, n_low=n + 8, protected_p=0, pyramid_n_min=0, fp16_window_w=W)
        eng = ConfKVEngine(cfg, ModelShape(L, H, D, 64, num_kv_heads=Hkv), quantize=quantize, batch=B,
                           capacity=n + 16)
        eng.begin_prefill(n)
        scale = float(rng.choice([0.1, 1.0, 4.0]))
        kv = torch.from_numpy((scale * rng.standard_normal((2, L, B, n, Hkv, D))).astype(np.float16))
        eng.prefill(kv[0], kv[1])
        if quantize:
            # one step demotes every entry with step <= 1 - W (a bulk segment), appends one entry
            for layer in range(L):
                eng.stage_rows(layer, np.full((B, H, n), 1.0 / n))
            z = torch.zeros((L, B, Hkv, D), dtype=torch.half)
            eng.step(torch.zeros((B, 64)), z, z, step=1)
            eng.records()
        q = torch.from_numpy((rng.standard_normal((L, B, H, D)) * float(rng.choice([0.5, 1.0, 3.0]))).astype(np.float16))
        out, w = eng.attend_layers(q, weights=True)
        out, w = out.cpu().numpy(), w.cpu().numpy()
        for layer in range(L):
            for b in range(B):
                st = eng.read_cache(layer, b)
                m = st["valid_len"]
                o_ref, w_ref = _naive(q[layer, b].float().numpy(), st["keys"], st["values"], G)
                eo = np.abs(out[layer, b] - o_ref).max(axis=1) / np.abs(o_ref).max(axis=1).clip(1e-30)
                ew = np.abs(w[layer, b, :, :m] - w_ref).max(axis=1) / w_ref.max(axis=1)
                worst_o, worst_w = max(worst_o, float(eo.max())), max(worst_w, float(ew.max()))
                assert eo.max() < 1e-3 and ew.max() < 1e-3, (it, D, G, n, layer, b, eo.max(), ew.max())
                cases += 1
        eng.close()
    assert cases >= 1000
    print(f"tiled vs naive ({'int8' if quantize else 'fp16'}): {cases} cases, worst rel out {worst_o:.2e}, "
          f"weights {worst_w:.2e}")


def test_int8_roundtrip_1e6():
    rng = np.random.default_rng(653)
    Hkv, D, n, W = 8, 128, 600, 64
    cfg = PolicyConfig(n_high=n + 8, n_low=n + 8, protected_p=0, pyramid_n_min=0, fp16_window_w=W)
    eng = ConfKVEngine(cfg, ModelShape(1, Hkv, D, 64), quantize=True, batch=1, capacity=n + 16)
    eng.begin_prefill(n)
    # per-channel magnitudes over 10 decades, exact zeros, fp16 subnormals
    chan = np.exp(rng.uniform(np.log(1e-6), np.log(1e4), size=(2, 1, Hkv, D)))
    x = np.clip(rng.standard_normal((2, n, Hkv, D)) * chan, -60000, 60000).astype(np.float16)
    x[:, :, 0, :4] = 0
    x[:, ::7, 1, 5] = np.float16(6e-8)
    eng.prefill(torch.from_numpy(x[0])[None, None], torch.from_numpy(x[1])[None, None])
    eng.stage_rows(0, np.full((1, Hkv, n), 1.0 / n))
    z = torch.zeros((1, 1, Hkv, D), dtype=torch.half)
    eng.step(torch.zeros((1, 64)), z, z, step=1)
    rec = eng.records()[0]
    st = eng.read_cache(0, 0)
    m = rec.int8[0]
    assert m == n + 2 - W   # prefill steps pos - n <= 1 - W  <=>  pos <= n + 1 - W
    total = 0
    for side, key, scales in ((0, "keys", "seg_k_scale"), (1, "values", "seg_v_scale")):
        xs = x[side, :m].astype(np.float32)
        codes, scale = O.quantize_lanes(xs)
        assert np.array_equal(st[scales][0], scale)
        assert np.array_equal(st["k_codes" if side == 0 else "v_codes"][:m], codes)
        xhat = st[key][:m]
        # |x - code*scale| <= scale/2 up to the fp32 rounding of x/scale and code*scale
        # (<= 127 * scale * 2^-23 each)
        assert np.all(np.abs(xs - xhat) <= scale[None] * (0.5 + 127 * 2.0**-22))
        total += xs.size
    assert total >= 10**6
    eng.close()
