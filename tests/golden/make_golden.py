"""Generate the golden fixtures that pin `oracle/` to the real reference.

Run in the build container (the only place `/root/reference` exists):

    python tests/golden/make_golden.py [--reference /root/reference/pkg/src]

It imports the UNMODIFIED reference package `confkv`, drives it on the seeded
inputs of `oracle/scenarios.py` and writes:

- `confidence.json`  — features / tier / argmax for seeded and edge logit rows
- `engine_<name>.npz` + `engine_<name>.json` — per-step StepRecords, attention
  outputs, kept old-index sets, and the final per-layer cache state
- `rng.json` — SplitMix64 draws, pinning `oracle.confkv_oracle.splitmix_normal`

GQA scenarios run the reference on K/V repeated across each query-head group
(the reference is MHA-only); the stored state keeps one copy per KV head after
asserting the copies are identical.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

from oracle import scenarios as S  # noqa: E402
from oracle.confkv_oracle import mix_u64, splitmix_normal  # noqa: E402

CONF_VOCABS = [2, 3, 64, 1000, 50257, 128256]
IO_SCENARIOS = ("int8_mha", "fp16_mha")   # MHA: the reference's snapshot heads = the engine's KV heads
CONF_ROWS = 6


def _ref(path):
    sys.path.insert(0, path)
    import confkv  # noqa: F401
    from confkv import attention, config, confidence, policy, rng
    return attention, config, confidence, policy, rng


def gen_rng(rng_mod):
    out = []
    for seed in (0, 1, 12345, 2**63 + 5):
        draws = rng_mod.SeededRng(seed).normal(7)
        mine = splitmix_normal(seed, 7)
        assert np.array_equal(draws, mine), "splitmix_normal diverges from rng.SeededRng.normal"
        out.append({"seed": seed, "normal7": [float(x) for x in draws]})
    for parts in ((1, 2, 3), (2**64 - 1, 0), (7,)):
        assert rng_mod.mix_u64(*parts) == mix_u64(*parts)
        out.append({"mix": list(parts), "value": rng_mod.mix_u64(*parts)})
    return out


def gen_confidence(conf_mod):
    rows = []
    for V in CONF_VOCABS:
        cases = [("seeded", t, S.step_logits(1000 + V, t, V)) for t in range(1, CONF_ROWS + 1)]
        cases += [("special", i, x) for i, x in enumerate(S.special_logits(V))]
        for kind, idx, logits in cases:
            for temp in (None, 0.7):
                x = logits if temp is None else np.asarray(logits, np.float64) / temp
                p = conf_mod.stable_softmax(x)
                f = conf_mod.confidence_score(p, (0.4, 0.3, 0.3))
                rows.append({
                    "V": V, "kind": kind, "idx": idx, "temperature": temp,
                    "digest": S.digest(logits),
                    "entropy_norm": f.entropy_norm, "margin": f.margin,
                    "margin_sig": f.margin_sig, "top_prob": f.top_prob, "score": f.score,
                    "tier": conf_mod.select_budget(f.score, 128, 256, 0.7),
                    "argmax": int(np.argmax(p)),
                })
    return rows


def gen_engine(name, spec, mods, outdir: Path):
    attention, config, confidence, policy, rng = mods
    L, H, Hkv, D, V = spec["L"], spec["H"], spec["Hkv"], spec["D"], spec["V"]
    G = H // Hkv
    cfg = config.PolicyConfig(**spec["cfg"])
    eng = policy.ConfKVEngine(cfg, config.ModelShape(L, H, D, V), quantize=spec["quantize"])
    seed = spec["seed"]
    eng.begin_prefill(spec["prefill"])
    for layer in range(L):
        k, v = S.scenario_prefill_kv(spec, seed, layer)
        for pos in range(spec["prefill"]):
            eng.append_prefill(layer, np.repeat(k[pos], G, 0), np.repeat(v[pos], G, 0), pos)

    records, outs, kept_flat, kept_len, rec_objs = [], [], [], [], []
    for t in range(1, spec["steps"] + 1):
        rows, step_out, before = [], [], []
        for layer, cache in enumerate(eng.caches):
            q = S.scenario_q(spec, seed, t, layer)
            o, w = attention.tiled_attention(q, cache, cfg.block_size_b)
            rows.append(w)
            step_out.append(o)
            before.append(cache.positions[: cache.valid_len].copy())
        new_kv = []
        for layer in range(L):
            k, v = S.step_kv(seed, t, layer, Hkv, D)
            new_kv.append((np.repeat(k, G, 0), np.repeat(v, G, 0)))
        rec_obj = eng.step(S.step_logits(seed, t, V), rows, new_kv, t)
        rec_objs.append(rec_obj)
        rec = rec_obj.to_dict()
        if cfg.sampling_mode != "greedy":
            rec["token"] = -1   # temperature sampling is outside the GPU path's scope
        records.append(rec)
        outs.append(np.stack(step_out))
        for layer, cache in enumerate(eng.caches):
            after = cache.positions[: rec["len_post"][layer]]
            kept = np.nonzero(np.isin(before[layer], after))[0]
            assert kept.shape[0] == rec["len_post"][layer]
            kept_flat.append(kept)
            kept_len.append(kept.shape[0])

    state = {}
    for layer, c in enumerate(eng.caches):
        n = c.valid_len
        sl = slice(0, None, G)  # one copy per KV head
        for arr in (c.keys, c.values, c.k_codes, c.v_codes):
            rep = arr[:n].reshape(n, Hkv, G, D)
            assert (rep == rep[:, :, :1, :]).all(), "replicated heads diverged"
        pre = f"l{layer}_"
        state[pre + "n"] = np.array(n)
        state[pre + "positions"] = c.positions[:n]
        state[pre + "steps"] = c.steps[:n]
        state[pre + "ema"] = c.ema[:n]
        state[pre + "seen"] = c.seen[:n]
        state[pre + "segment_of"] = c.segment_of[:n]
        # K/V inputs are fp16-representable: fp16 storage is exact and halves the fixture
        kv = c.keys[:n][:, sl]
        assert np.array_equal(kv.astype(np.float16).astype(np.float32), kv)
        state[pre + "keys"] = kv.astype(np.float16)
        state[pre + "values"] = c.values[:n][:, sl].astype(np.float16)
        state[pre + "k_codes"] = c.k_codes[:n][:, sl]
        state[pre + "v_codes"] = c.v_codes[:n][:, sl]
        state[pre + "seg_k_scale"] = (np.stack([s.k_scale[sl] for s in c.segments])
                                      if c.segments else np.zeros((0, Hkv, D), np.float32))
        state[pre + "seg_v_scale"] = (np.stack([s.v_scale[sl] for s in c.segments])
                                      if c.segments else np.zeros((0, Hkv, D), np.float32))
        state[pre + "seg_count"] = np.array([s.member_count for s in c.segments], np.int64)

    if name in IO_SCENARIOS:
        # F3 fixtures: the reference's own JSONL trace, TraceSummary and CKVS snapshots
        analysis = __import__("confkv.analysis", fromlist=["summarize_trace"])
        with open(outdir / f"trace_{name}.jsonl", "w") as f:
            for r in rec_objs:
                f.write(json.dumps(r.to_dict()) + "\n")
        with open(outdir / f"summary_{name}.json", "w") as f:
            json.dump(analysis.summarize_trace(rec_objs).to_dict(), f)
        for layer, c in enumerate(eng.caches):
            c.write_snapshot(outdir / f"snap_{name}_l{layer}.ckvs", layer)

    sampled = [t for t in range(len(outs)) if t % 20 == 0]
    np.savez_compressed(outdir / f"engine_{name}.npz", out_steps=np.array(sampled),
                        outs=np.stack([outs[t] for t in sampled]),
                        kept_flat=np.concatenate(kept_flat), kept_len=np.array(kept_len), **state)
    with open(outdir / f"engine_{name}.json", "w") as f:
        json.dump({"spec": spec, "config_json": cfg.to_json(), "config_hash": cfg.config_hash(),
                   "records": records,
                   "out_digests": [S.digest(o) for o in outs]}, f)
    return len(records)


BASELINE_SCENARIO = "int8_mha"   # inputs and config of this scenario, run FP16 (baselines never quantize)
BASELINE_RUNS = [("full", {}), ("sliding", {"window": 60}), ("heavy_hitter", {"cap": 72}),
                 ("matched", {"mode": "random"}), ("matched", {"mode": "recency_only"}),
                 ("matched", {"mode": "attention_only"})]


def baseline_tag(kind, kw):
    return kind if kind != "matched" else f"matched_{kw['mode']}"


def gen_baselines(mods, outdir: Path):
    """F4 fixtures: the reference's comparison policies (baselines.py) on one scenario's inputs;
    the matched-rate runs replay the eviction schedule recorded by a ConfKVEngine run
    (record_schedule=True) on the same inputs."""
    attention, config, confidence, policy, rng = mods
    baselines = __import__("confkv.baselines", fromlist=["SlidingWindowPolicy"])
    spec = S.SCENARIOS[BASELINE_SCENARIO]
    L, H, Hkv, D, V, seed = spec["L"], spec["H"], spec["Hkv"], spec["D"], spec["V"], spec["seed"]
    G = H // Hkv
    cfg = config.PolicyConfig(**spec["cfg"])
    shape = config.ModelShape(L, H, D, V)

    def drive(pol):
        pol.begin_prefill(spec["prefill"])
        for layer in range(L):
            k, v = S.scenario_prefill_kv(spec, seed, layer)
            for pos in range(spec["prefill"]):
                pol.append_prefill(layer, np.repeat(k[pos], G, 0), np.repeat(v[pos], G, 0), pos)
        recs, kept_flat = [], []
        for t in range(1, spec["steps"] + 1):
            rows, before = [], []
            for layer, cache in enumerate(pol.caches):
                o, w = attention.tiled_attention(S.scenario_q(spec, seed, t, layer), cache, cfg.block_size_b)
                rows.append(w)
                before.append(cache.positions[: cache.valid_len].copy())
            new_kv = []
            for layer in range(L):
                k, v = S.step_kv(seed, t, layer, Hkv, D)
                new_kv.append((np.repeat(k, G, 0), np.repeat(v, G, 0)))
            rec = pol.step(S.step_logits(seed, t, V), rows, new_kv, t).to_dict()
            recs.append(rec)
            for layer, cache in enumerate(pol.caches):
                after = cache.positions[: rec["len_post"][layer]]
                kept_flat.append(np.nonzero(np.isin(before[layer], after))[0])
        return recs, kept_flat

    src = policy.ConfKVEngine(cfg, shape, quantize=False, record_schedule=True)
    drive(src)
    schedule = [(e.step, e.layer, e.evict_count) for e in src.schedule]
    for kind, kw in BASELINE_RUNS:
        if kind == "full":
            pol = baselines.FullCachePolicy(cfg, shape)
        elif kind == "sliding":
            pol = baselines.SlidingWindowPolicy(cfg, shape, window=kw["window"])
        elif kind == "heavy_hitter":
            pol = baselines.HeavyHitterPolicy(cfg, shape, cap=kw["cap"])
        else:
            pol = baselines.MatchedRatePolicy(cfg, shape, list(src.schedule), kw["mode"])
        recs, kept_flat = drive(pol)
        tag = baseline_tag(kind, kw)
        state = {"kept_flat": np.concatenate(kept_flat), "kept_len": np.array([k.shape[0] for k in kept_flat])}
        for layer, c in enumerate(pol.caches):
            n = c.valid_len
            pre = f"l{layer}_"
            state[pre + "positions"] = c.positions[:n]
            state[pre + "steps"] = c.steps[:n]
            state[pre + "ema"] = c.ema[:n]
            state[pre + "seen"] = c.seen[:n]
            state[pre + "cum"] = c.aux[baselines.CUM_ATTENTION][:n] if baselines.CUM_ATTENTION in c.aux \
                else np.zeros(n)
        np.savez_compressed(outdir / f"baseline_{tag}.npz", **state)
        with open(outdir / f"baseline_{tag}.json", "w") as f:
            json.dump({"kind": kind, "kwargs": kw, "scenario": BASELINE_SCENARIO, "name": pol.name,
                       "schedule": schedule, "records": recs}, f)
        print(f"baseline_{tag}: {len(recs)} steps, evicted {sum(sum(r['evicted']) for r in recs)}")


RUN_DECODE_POLICIES = ("confkv", "confkv-int8", "confkv-l")
RUN_DECODE_SEED, RUN_DECODE_TRACES = 2026, 2


def gen_run_decode(ref_path: str, outdir: Path):
    """The reference's own driver protocol end to end: `retention_suite` needle traces
    (simulator.py:342-375) written with `SyntheticTrace.write_jsonl`, replayed by
    `run_decode` + `TraceDriver` (simulator.py:408-478) through the reference's policies
    (cli.py:82-88), StepRecord JSONL sinks and `needle_retained` saved. The GPU test drives
    the B200 engine through a restatement of the same loop and must reproduce the JSONL."""
    sys.path.insert(0, ref_path)
    from confkv.config import ModelShape, PolicyConfig
    from confkv.policy import ConfKVEngine
    from confkv.simulator import TraceDriver, retention_suite, run_decode
    cfg = PolicyConfig()
    traces = retention_suite(RUN_DECODE_SEED, RUN_DECODE_TRACES, shape=ModelShape(num_layers=3))
    meta = {"seed": RUN_DECODE_SEED, "policies": list(RUN_DECODE_POLICIES), "runs": []}
    for k, trace in enumerate(traces):
        trace.write_jsonl(outdir / f"rundecode_trace{k}.jsonl")
        for name in RUN_DECODE_POLICIES:
            pol = ConfKVEngine(cfg.replace(pyramid_enabled=name == "confkv-l"), trace.shape,
                               quantize=name != "confkv")
            path = outdir / f"rundecode_{name}_trace{k}.jsonl"
            with open(path, "w") as sink:
                res = run_decode(pol, TraceDriver(trace), len(trace), sink=sink)
            meta["runs"].append({"trace": k, "policy": name, "steps": len(trace),
                                 "needle_retained": res.needle_retained, "jsonl": path.name})
            print(f"rundecode {name} trace{k}: {len(trace)} steps, needle retained {res.needle_retained}")
    with open(outdir / "rundecode.json", "w") as f:
        json.dump(meta, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default=os.environ.get("CONFKV_REF", "/root/reference/pkg/src"))
    ap.add_argument("--out", default=str(HERE))
    ap.add_argument("--only", default="", help="comma-separated scenario names (default: all)")
    ap.add_argument("--baselines", action="store_true", help="only the F4 comparison-policy fixtures")
    ap.add_argument("--run-decode", action="store_true", help="only the run_decode / TraceDriver fixtures")
    args = ap.parse_args()
    mods = _ref(args.reference)
    out = Path(args.out)
    if args.run_decode:
        gen_run_decode(args.reference, out)
        return
    if not args.only:
        with open(out / "rng.json", "w") as f:
            json.dump(gen_rng(mods[4]), f, indent=1)
        with open(out / "confidence.json", "w") as f:
            json.dump(gen_confidence(mods[2]), f)
    if args.baselines:
        gen_baselines(mods, out)
        return
    only = set(args.only.split(",")) if args.only else None
    for name, spec in S.SCENARIOS.items():
        if only and name not in only:
            continue
        n = gen_engine(name, spec, mods, out)
        print(f"engine_{name}: {n} steps")


if __name__ == "__main__":
    main()
