"""INT8 storage on the device: lossy-segment codes in place in the fp16 slot rows,
single-entry segments kept as their fp16 rows (codes / scales synthesised), the lossy scale
pool sized by max_segments. Checked against the oracle (pinned to the reference) and the
reference quantizer (quantizer.py:16-34, restated as oracle.quantize_lanes)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import confkv_oracle as O  # noqa: E402
from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402
from tests.gpu_driver import compare_attention, compare_cache  # noqa: E402


def _all_fp16():
    """Every finite fp16 value (63,488 of them), padded with zeros to a multiple of 1,024."""
    u = np.arange(65536, dtype=np.uint16).view(np.float16)
    f = u[np.isfinite(u)].astype(np.float32)
    return np.concatenate([f, np.zeros(-f.size % 1024, np.float32)])


def test_single_entry_segments_every_fp16_value():
    """Decode-built single-entry segments (the reference's steady state): every finite fp16
    value demoted alone. ckv_read_cache's codes and scale rows (synthesised from the resident
    fp16 row) must equal quantize_segment of that one entry, and its dequantised view
    code * scale; K2 reads x itself, which differs from code * scale by <= 1 fp32 ulp."""
    vals = _all_fp16().reshape(-1, 8, 128)          # [62, Hkv=8, D=128] entries
    m = vals.shape[0]
    cfg = PolicyConfig(n_high=200, n_low=200, protected_p=0, pyramid_n_min=0, fp16_window_w=1)
    eng = ConfKVEngine(cfg, ModelShape(1, 8, 128, 64), quantize=True, batch=1, capacity=256)
    eng.begin_prefill(1)
    z = torch.zeros((1, 1, 1, 8, 128), dtype=torch.half)
    eng.prefill(z, z)
    for t in range(1, m + 3):
        eng.stage_rows(0, np.full((1, 8, t), 1.0 / t))
        kv = vals[t - 1] if t <= m else np.zeros((8, 128), np.float32)
        k = torch.from_numpy(kv).half()[None, None]
        v = torch.from_numpy(-kv).half()[None, None]
        eng.step(torch.zeros((1, 64)), k, v, step=t)
        eng.records()
    st = eng.read_cache(0, 0)
    ulp_off = 0
    for i in range(m):
        j = i + 1   # storage: the prefill entry, then the step-t entry at j = t (holds vals[t - 1])
        for side, key, codes, scale, sign in (("k", "keys", "k_codes", "seg_k_scale", 1.0),
                                              ("v", "values", "v_codes", "seg_v_scale", -1.0)):
            x = (sign * vals[i]).astype(np.float32)
            c_ref, s_ref = O.quantize_lanes(x[None])
            sg = st["segment_of"][j]
            assert st["seg_count"][sg] == 1
            assert np.array_equal(st[codes][j], c_ref[0]), (i, side)
            assert np.array_equal(st[scale][sg], s_ref), (i, side)
            xh = (c_ref[0].astype(np.float32) * s_ref)
            assert np.array_equal(st[key][j], xh), (i, side)
            d = xh != x
            ulp_off += int(d.sum())
            assert np.all(np.abs(xh[d] - x[d]) <= np.spacing(np.abs(x[d]))), (i, side)
    # 214 of the 31,743 positive finite magnitudes round off by one ulp, in K and in V, +/-
    assert ulp_off == 4 * 214, ulp_off
    eng.close()


def _drive_jumps(eng, orc, L, H, Hkv, D, V, steps, seed):
    rng = np.random.default_rng(seed)
    worst = 0.0
    for t in steps:
        q = rng.standard_normal((L, 1, H, D)).astype(np.float16).astype(np.float32)
        out, w = eng.attend_layers(torch.from_numpy(q), weights=True)
        out, w = out.cpu().numpy(), w.cpu().numpy()
        rows = []
        for layer in range(L):
            o_ref, _ = orc.attend(layer, q[layer, 0])
            worst = max(worst, compare_attention(out[layer, 0][None], o_ref[None], f"t={t} l={layer}"))
            rows.append(w[layer, 0, :, : orc.caches[layer].n].astype(np.float64))
        kn = rng.standard_normal((L, 1, Hkv, D)).astype(np.float16).astype(np.float32)
        vn = rng.standard_normal((L, 1, Hkv, D)).astype(np.float16).astype(np.float32)
        logits = rng.standard_normal((1, V)).astype(np.float32).astype(np.float64)
        eng.step(torch.from_numpy(logits).float(), torch.from_numpy(kn), torch.from_numpy(vn), step=t)
        rec = orc.step(logits[0], rows, [(kn[layer, 0], vn[layer, 0]) for layer in range(L)], t)
        g = eng.records()[0]
        for key in ("len_pre", "len_post", "evicted", "int8", "memory_bytes", "budget"):
            assert getattr(g, key) == rec[key], (t, key, getattr(g, key), rec[key])
        for layer in range(L):
            compare_cache(eng.read_cache(layer, 0), orc.caches[layer], f"t={t} l={layer}")
    return worst


def test_step_jump_turns_single_entry_segments_lossy():
    """Steps 1..6 demote one entry each (single-entry segments, fp16 rows); the jump to step 20
    ages the step-4..6 entries at once: a lossy segment forms after the single-entry ones, so every INT8
    entry is read as codes from then on (the earlier single-entry segments get lossy-pool ids,
    scale rows and in-place codes). State, records and attention against the oracle."""
    L, H, Hkv, D, V = 2, 8, 2, 128, 64
    cfg = PolicyConfig(n_high=200, n_low=200, protected_p=4, pyramid_n_min=4, fp16_window_w=3)
    eng = ConfKVEngine(cfg, ModelShape(L, H, D, V, num_kv_heads=Hkv), quantize=True, batch=1, capacity=256)
    orc = O.OracleEngine(cfg, L, H, D, V, quantize=True, kv_heads=Hkv)
    rng = np.random.default_rng(5)
    pf = 2
    kv = rng.standard_normal((2, L, pf, Hkv, D)).astype(np.float16).astype(np.float32)
    eng.begin_prefill(pf)
    orc.begin_prefill(pf)
    eng.prefill(torch.from_numpy(kv[0][:, None]), torch.from_numpy(kv[1][:, None]))
    for layer in range(L):
        for p in range(pf):
            orc.append_prefill(layer, kv[0, layer, p], kv[1, layer, p], p)
    worst = _drive_jumps(eng, orc, L, H, Hkv, D, V, [1, 2, 3, 4, 5, 6, 20, 21, 22], seed=9)
    assert worst < 1e-3
    st = eng.read_cache(0, 0)
    assert st["num_segments"] > 1 and max(st["seg_count"]) > 1
    eng.close()


def test_lossy_pool_exhaustion_raises():
    """Two lossy segments with max_segments=1: reported (RuntimeError), never truncated."""
    L, H, D, V = 1, 2, 16, 64
    cfg = PolicyConfig(n_high=100, n_low=100, protected_p=0, pyramid_n_min=0, fp16_window_w=50)
    eng = ConfKVEngine(cfg, ModelShape(L, H, D, V), quantize=True, batch=1, capacity=128, max_segments=1)
    eng.begin_prefill(10)
    kv = torch.randn((1, 1, 10, H, D)).half()
    eng.prefill(kv, kv)
    z = torch.zeros((1, 1, H, D), dtype=torch.half)
    # step 100 ages the prefill + steps 1-3 (lossy segment 1), step 300 steps 100-102 (lossy 2)
    for t in (1, 2, 3, 100, 101, 102, 300):
        n = eng.caches[0].valid_len
        eng.stage_rows(0, np.full((1, H, n), 1.0 / n))
        eng.step(torch.zeros((1, V)), z, z, step=t)
        if t != 300:
            eng.records()
    with pytest.raises(RuntimeError, match="capacity exhausted"):
        eng.records()
    eng.close()


def test_int8_footprint_is_the_fp16_slot_pool():
    """INT8 adds no per-entry storage over FP16 (codes live in the fp16 slot rows, single-entry
    segments have no scale rows): device bytes within 5% of the FP16 engine's at Llama shape."""
    shape = ModelShape(2, 32, 128, 1000, num_kv_heads=8)
    cfg = PolicyConfig(n_high=4096, n_low=4096, protected_p=64, alpha=0.7, fp16_window_w=256, pyramid_n_min=96)
    a = ConfKVEngine(cfg, shape, quantize=True, batch=2, capacity=4098)
    b = ConfKVEngine(cfg, shape, quantize=False, batch=2, capacity=4098)
    assert a.device_bytes <= 1.05 * b.device_bytes, (a.device_bytes, b.device_bytes)
    a.close()
    b.close()


def test_prefill_past_capacity():
    """a prefill that does not fit raises before the first step; after stepping
    began, an overflowing chunk is reported by every later step's records (sticky)."""
    cfg = PolicyConfig(n_high=20, n_low=20, protected_p=4, pyramid_n_min=4)
    eng = ConfKVEngine(cfg, ModelShape(1, 2, 16, 64), batch=1, capacity=24)
    eng.begin_prefill(30)
    kv = torch.zeros((1, 1, 12, 2, 16), dtype=torch.half)
    eng.prefill(kv, kv)
    eng.prefill(kv, kv)
    with pytest.raises(ValueError, match="capacity"):
        eng.prefill(kv, kv)    # 36 > 24 before any step
    z = torch.zeros((1, 1, 2, 16), dtype=torch.half)
    eng.stage_rows(0, np.full((1, 2, 24), 1.0 / 24))
    eng.step(torch.zeros((1, 64)), z, z, step=1)
    eng.records()
    eng.prefill(kv, kv)        # 21 + 12 > 24: dropped on the device
    n = eng.caches[0].valid_len
    eng.stage_rows(0, np.full((1, 2, n), 1.0 / n))
    eng.step(torch.zeros((1, 64)), z, z, step=2)
    with pytest.raises(RuntimeError, match="capacity exhausted"):
        eng.records()
    eng.close()


def test_stage_rows_length_mismatch():
    """rows shorter / longer than valid_len are a ValueError (cache.py:164-167),
    for the batched tensor and for ragged per-sequence lists."""
    cfg = PolicyConfig(n_high=20, n_low=20, protected_p=4, pyramid_n_min=4)
    eng = ConfKVEngine(cfg, ModelShape(1, 2, 16, 64), batch=2, capacity=24)
    eng.begin_prefill(10)
    kv = torch.zeros((1, 2, 10, 2, 16), dtype=torch.half)
    eng.prefill(kv, kv)
    z = torch.zeros((1, 2, 2, 16), dtype=torch.half)
    for rows in (np.full((2, 2, 9), 1.0 / 9), [np.full((2, 10), 0.1), np.full((2, 11), 1.0 / 11)]):
        eng.stage_rows(0, rows)
        eng.step(torch.zeros((2, 64)), z, z, step=eng._next_t)
        with pytest.raises(ValueError, match="valid_len"):
            eng.records()
    eng.close()
