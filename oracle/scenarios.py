"""Seeded synthetic inputs + scenario specs shared by the golden generator,
the CPU oracle tests and the GPU parity tests. TEST INFRASTRUCTURE ONLY.

Every input is a pure function of (scenario seed, stream tag, step, layer)
through SplitMix64 (`confkv_oracle.mix_u64` / `splitmix_normal`, restating
the reference's `rng.py`), so fixtures store outputs plus input digests, not
the inputs. K/V/q values are rounded to fp16 (the GPU stores fp16), logits to
fp32 (the GPU consumes fp32 logits): both sides then see identical values.
"""

from __future__ import annotations

import hashlib

import numpy as np

from .confkv_oracle import mix_u64, splitmix_normal

TAG_Q, TAG_K, TAG_V, TAG_LOGIT, TAG_GAIN, TAG_PREFILL, TAG_NEEDLE = 0x71, 0x6B, 0x76, 0x6C, 0x67, 0x70, 0x6E


def fp16_normal(seed: int, shape) -> np.ndarray:
    n = int(np.prod(shape))
    return splitmix_normal(seed, n).astype(np.float16).astype(np.float32).reshape(shape)


def step_logits(seed: int, t: int, vocab: int, gains=(8.0, 0.5)) -> np.ndarray:
    """gain * N(0,1), fp32-representable. Gain is gains[0] on 3 of 4 steps
    (peaky -> confident) and gains[1] otherwise (flat -> uncertain)."""
    g = gains[0] if (mix_u64(seed, TAG_GAIN, t) & 3) != 0 else gains[1]
    return (g * splitmix_normal(mix_u64(seed, TAG_LOGIT, t), vocab)).astype(np.float32).astype(np.float64)


def step_q(seed, t, layer, hq, d):
    return fp16_normal(mix_u64(seed, TAG_Q, t, layer), (hq, d))


def step_kv(seed, t, layer, hkv, d):
    return (fp16_normal(mix_u64(seed, TAG_K, t, layer), (hkv, d)),
            fp16_normal(mix_u64(seed, TAG_V, t, layer), (hkv, d)))


def prefill_kv(seed, layer, n, hkv, d):
    """[n, Hkv, D] K and V for positions 0..n-1 of one layer."""
    k = fp16_normal(mix_u64(seed, TAG_PREFILL, 0, layer), (n, hkv, d))
    v = fp16_normal(mix_u64(seed, TAG_PREFILL, 1, layer), (n, hkv, d))
    return k, v


def needle_dir(seed, layer, hkv, d):
    """Unit needle direction per KV head [Hkv, D] (fp64)."""
    u = splitmix_normal(mix_u64(seed, TAG_NEEDLE, layer), hkv * d).reshape(hkv, d)
    return u / np.linalg.norm(u, axis=1, keepdims=True)


def scenario_q(spec, seed, t, layer):
    """step_q, plus for needle scenarios a component `q_gain * u` along the layer's needle
    direction (every query head of the KV head's group), fp16-rounded: the planted needle
    key then draws a large attention mass at every step."""
    q = step_q(seed, t, layer, spec["H"], spec["D"])
    nd = spec.get("needle")
    if nd is None:
        return q
    u = np.repeat(needle_dir(seed, layer, spec["Hkv"], spec["D"]), spec["H"] // spec["Hkv"], axis=0)
    return (q + nd["q_gain"] * u).astype(np.float16).astype(np.float32)


def scenario_prefill_kv(spec, seed, layer):
    """prefill_kv, with the needle key `k_gain * u` planted at the needle position."""
    k, v = prefill_kv(seed, layer, spec["prefill"], spec["Hkv"], spec["D"])
    nd = spec.get("needle")
    if nd is not None:
        k[nd["pos"]] = (nd["k_gain"] * needle_dir(seed, layer, spec["Hkv"], spec["D"])
                        ).astype(np.float16).astype(np.float32)
    return k, v


def special_logits(vocab: int) -> list[np.ndarray]:
    """Edge rows for confidence: all-equal, tied top-2, runner-up underflow
    (p2 below the 1e-12 floor), huge offsets (shift invariance), and a
    clear winner at the last index (argmax tie rules / scan tails)."""
    rows = [np.zeros(vocab)]
    r = np.linspace(-3.0, 3.0, vocab)
    r[vocab // 3] = r[-1] = 5.0           # exact tie for the top -> margin 0, argmax = vocab//3
    rows.append(r)
    r = np.zeros(vocab)
    r[1] = 80.0                            # p2 = e^-80 < 1e-12 -> floored
    rows.append(r)
    rows.append(np.full(vocab, 1000.0) + np.arange(vocab) % 7)
    r = -np.arange(vocab, dtype=np.float64) / vocab
    r[-1] = 2.0
    rows.append(r)
    return [x.astype(np.float32).astype(np.float64) for x in rows]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


# Engine scenarios. `cfg` holds PolicyConfig fields; `quantize` is the
# reference's ConfKVEngine(quantize=...) flag (cli.py:83-88: confkv /
# confkv-int8 / confkv-l).
SCENARIOS: dict[str, dict] = {
    # defaults (wikitext column), FP16 only, MHA
    "fp16_mha": dict(L=2, H=4, Hkv=4, D=16, V=64, prefill=120, steps=160, quantize=False,
                     cfg={}, seed=11),
    # INT8 window with a bulk first segment, MHA, small budgets
    "int8_mha": dict(L=3, H=4, Hkv=4, D=32, V=257, prefill=80, steps=160, quantize=True,
                     cfg=dict(n_high=48, n_low=96, protected_p=16, pyramid_n_min=32,
                              fp16_window_w=24, alpha=0.7), seed=22),
    # GQA (group 4) + pyramid + INT8 (confkv-l)
    "pyramid_gqa": dict(L=4, H=8, Hkv=2, D=64, V=1000, prefill=100, steps=140, quantize=True,
                        cfg=dict(n_high=64, n_low=128, protected_p=16, pyramid_n_min=40,
                                 fp16_window_w=32, pyramid_enabled=True), seed=33),
    # edge knobs: P=0, W=0 (everything ages at once), alpha=1 (attention only), lambda=0
    "edge_p0_w0": dict(L=2, H=2, Hkv=2, D=16, V=50, prefill=40, steps=90, quantize=True,
                       cfg=dict(n_high=20, n_low=30, protected_p=0, pyramid_n_min=8,
                                fp16_window_w=0, alpha=1.0, ema_lambda=0.0), seed=44),
    # Llama-like head dim 128, GQA group 4, several 512-entry splits, FP16 only
    "fp16_d128_long": dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=1100, steps=24, quantize=False,
                           cfg=dict(n_high=1060, n_low=1100, protected_p=64, pyramid_n_min=96,
                                    alpha=0.7), seed=66),
    # same with the INT8 window: one bulk segment, singletons, a mixed boundary split
    "int8_d128_long": dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=1100, steps=24, quantize=True,
                           cfg=dict(n_high=1060, n_low=1100, protected_p=64, pyramid_n_min=96,
                                    alpha=0.7, fp16_window_w=600), seed=77),
    # small window: one bulk segment spans whole 512-entry splits (integer tensor-core path)
    "int8_bulk_d128": dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=1100, steps=24, quantize=True,
                           cfg=dict(n_high=1060, n_low=1100, protected_p=64, pyramid_n_min=96,
                                    alpha=0.7, fp16_window_w=64), seed=88),
    # recency only (alpha=0), lambda=1, GQA group 2, temperature-scaled confidence
    "edge_alpha0_temp": dict(L=2, H=4, Hkv=2, D=32, V=128, prefill=64, steps=100, quantize=False,
                             cfg=dict(n_high=40, n_low=56, protected_p=8, pyramid_n_min=16,
                                      alpha=0.0, ema_lambda=1.0, sampling_mode="temperature",
                                      temperature=0.7), seed=55),
    # Qwen-like GQA group 5 (Hq/Hkv = 40/8 scaled down), D=128, INT8 with a bulk segment
    "gqa5_int8_d128": dict(L=2, H=10, Hkv=2, D=128, V=900, prefill=1100, steps=24, quantize=True,
                           cfg=dict(n_high=1060, n_low=1100, protected_p=64, pyramid_n_min=96,
                                    alpha=0.7, fp16_window_w=64), seed=111),
    # GQA group 8, D=64, FP16 + INT8 window, pyramid budgets
    "gqa8_int8_d64": dict(L=3, H=16, Hkv=2, D=64, V=500, prefill=300, steps=60, quantize=True,
                          cfg=dict(n_high=200, n_low=280, protected_p=32, pyramid_n_min=96,
                                   fp16_window_w=48, pyramid_enabled=True), seed=122),
    # K2 split geometry: budget a multiple of 512, so every step attends budget + 1 entries and
    # the 1-entry tail split is read by the last full split (INT8: codes part + FP16 window;
    # FP16: one 513-entry split)
    "absorb_int8_d128": dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=1100, steps=16, quantize=True,
                             cfg=dict(n_high=1024, n_low=1024, protected_p=64, pyramid_n_min=96,
                                      alpha=0.7, fp16_window_w=64), seed=133),
    "absorb_fp16_d128": dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=600, steps=16, quantize=False,
                             cfg=dict(n_high=512, n_low=512, protected_p=64, pyramid_n_min=96,
                                      alpha=0.7), seed=144),
    # C1 at its real shape: GPT-2 small, L=12, H=12 (MHA), D=64, V=50,257,
    # 512-entry prefill, all 512 decode steps, FP16 cache, tau=0.7, 128/256, P=64, alpha=0.65,
    # lambda=0.9, W=128 (step 1 selects 512 -> 128/256 with the radix select)
    "gpt2_c1": dict(L=12, H=12, Hkv=12, D=64, V=50257, prefill=512, steps=512, quantize=False,
                    cfg=dict(n_high=128, n_low=256, protected_p=64, alpha=0.65, ema_lambda=0.9,
                             fp16_window_w=128), seed=1001),
    # C4: needle-in-a-haystack, 32K prefill, niah preset budgets (256/512, P=64, alpha=0.70,
    # W=256) with INT8: step 1 attends 32,768 entries, selects 32,768 -> 256/512 and demotes the
    # aged survivors into one bulk segment; the planted needle must survive (retention)
    "niah_32k": dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=32768, steps=8, quantize=True,
                     cfg=dict(n_high=256, n_low=512, protected_p=64, pyramid_n_min=96, alpha=0.70,
                              fp16_window_w=256),
                     needle=dict(pos=12345, q_gain=8.0, k_gain=16.0), seed=99),
}


def drive_oracle(name: str, cfg, engine_cls, capacity=64):
    """Run one scenario through the oracle exactly as make_golden.py drives the
    reference. Returns (records, per-step outs, per-(step, layer) kept arrays, engine)."""
    spec = SCENARIOS[name]
    L, H, Hkv, D, V, seed = spec["L"], spec["H"], spec["Hkv"], spec["D"], spec["V"], spec["seed"]
    eng = engine_cls(cfg, L, H, D, V, quantize=spec["quantize"], kv_heads=Hkv, capacity=capacity)
    eng.begin_prefill(spec["prefill"])
    for layer in range(L):
        k, v = scenario_prefill_kv(spec, seed, layer)
        for pos in range(spec["prefill"]):
            eng.append_prefill(layer, k[pos], v[pos], pos)
    records, outs, kept = [], [], []
    for t in range(1, spec["steps"] + 1):
        rows, step_out = [], []
        for layer in range(L):
            o, w = eng.attend(layer, scenario_q(spec, seed, t, layer))
            rows.append(w)
            step_out.append(o)
        new_kv = [step_kv(seed, t, layer, Hkv, D) for layer in range(L)]
        rec, kp = eng.step(step_logits(seed, t, V), rows, new_kv, t, return_kept=True)
        records.append(rec)
        outs.append(np.stack(step_out))
        kept.extend(kp)
    return records, outs, kept, eng
