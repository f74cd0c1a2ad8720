"""Drive the GPU engine and the CPU oracle side by side on the seeded
scenarios (oracle/scenarios.py). Test infrastructure.

Protocol: every step the GPU computes attention (fp32);
its normalised weights are handed to the oracle's `step` as the attention
rows, so the oracle's EMA, ranking, eviction and INT8 demotion run on exactly
the numbers the GPU's manager consumed. Kept sets, EMA bits, INT8 codes and
scales, positions, segment structure and the StepRecord integers must then
agree exactly; attention outputs are compared to the oracle's own fp64
attention with a 1e-3 relative tolerance; confidence features to 1e-9.
"""

from __future__ import annotations

import copy

import numpy as np
import torch

from oracle import confkv_oracle as O
from oracle import scenarios as S
from paper_2605_24786_b200.config import ModelShape, PolicyConfig
from paper_2605_24786_b200.engine import ConfKVEngine

ATTN_RTOL = 1e-3
CONF_RTOL = 1e-9


def seq_seed(spec, b):
    return spec["seed"] + 1000 * b


def compare_attention(out_gpu: np.ndarray, out_ref: np.ndarray, what: str):
    """Per (head) row: max |gpu - ref| <= ATTN_RTOL * max |ref row| (+ tiny floor)."""
    err = np.abs(out_gpu - out_ref).max(axis=-1)
    scale = np.abs(out_ref).max(axis=-1)
    bad = err > ATTN_RTOL * scale + 1e-7
    assert not bad.any(), f"{what}: attention mismatch, worst rel {float((err / (scale + 1e-30)).max()):.3e}"
    return float((err / (scale + 1e-30)).max())


def compare_cache(gpu: dict, ref: O.OracleCache, what: str):
    n = ref.n
    assert gpu["valid_len"] == n, f"{what}: valid_len {gpu['valid_len']} != {n}"
    assert np.array_equal(gpu["positions"], ref.pos[:n]), f"{what}: positions"
    assert np.array_equal(gpu["steps"], ref.step[:n]), f"{what}: steps"
    assert np.array_equal(gpu["ema"], ref.ema[:n]), f"{what}: ema bits"
    if "cum" in gpu:
        assert np.array_equal(gpu["cum"], ref.cum[:n]), f"{what}: cumulative attention bits"
    assert np.array_equal(gpu["seen"], ref.seen[:n]), f"{what}: seen"
    assert np.array_equal(gpu["segment_of"], ref.seg[:n]), f"{what}: segment ids"
    assert gpu["num_segments"] == len(ref.seg_count), f"{what}: segment count"
    q8 = ref.seg[:n] != O.HIGH
    assert np.array_equal(gpu["k_codes"][q8], ref.kc[:n][q8]), f"{what}: K codes"
    assert np.array_equal(gpu["v_codes"][q8], ref.vc[:n][q8]), f"{what}: V codes"
    if ref.seg_count:
        assert np.array_equal(gpu["seg_count"], np.array(ref.seg_count, np.int32)), f"{what}: members"
        assert np.array_equal(gpu["seg_k_scale"], np.stack(ref.seg_k)), f"{what}: K scales"
        assert np.array_equal(gpu["seg_v_scale"], np.stack(ref.seg_v)), f"{what}: V scales"
    kd, vd = ref.dequant_kv(0, n) if n else (ref.k[:0], ref.v[:0])
    assert np.array_equal(gpu["keys"], kd), f"{what}: dequantized K"
    assert np.array_equal(gpu["values"], vd), f"{what}: dequantized V"


def run_scenario(name: str, batch: int = 2, steps: int | None = None, check_every: int = 25,
                 use_gpu_rows: bool = True, on_step=None, on_end=None, make_engine=None, make_oracle=None,
                 production: bool = False, graph: bool = False, own_attention_trials: bool = False):
    """Returns a summary dict; asserts on any mismatch. on_step(t, records) after every
    step, on_end(engine) before the engine is closed. make_engine(cfg, shape, batch, cap) /
    make_oracle(cfg) swap in another policy (the F4 comparison policies).

    production: after the weights-dumping attention (the oracle's rows), the step itself runs
    the production path -- `step(q=...)`: attention without the weights dump (the WD=false
    combine), K1 forked beside it, K3/K4 with the kept-index map; graph=True replays it from
    one `capture_step` CUDA graph, as the bench does. The production path's staged head mean
    must equal the weights-dump path's bit for bit and its output must equal the dump path's
    output, so the oracle checks (fed the dumped weights) cover the production kernels.

    own_attention_trials: every step, a copy of each oracle is also stepped with its OWN fp64
    attention rows (the reference end to end) from the same pre-step state,
    and its kept sets are compared with the GPU's: the summary's kept_mismatch / kept_trials
    count the (step, sequence, layer) decisions where fp32 GPU attention and the reference's
    fp64 attention keep different entries (each trial starts from the synced state)."""
    spec = S.SCENARIOS[name]
    L, H, Hkv, D, V = spec["L"], spec["H"], spec["Hkv"], spec["D"], spec["V"]
    cfg = PolicyConfig(**spec["cfg"])
    shape = ModelShape(L, H, D, V, num_kv_heads=Hkv)
    nsteps = steps or spec["steps"]
    cap = max(spec["prefill"], max(cfg.n_low, cfg.n_high)) + 2
    if make_engine is None:
        eng = ConfKVEngine(cfg, shape, quantize=spec["quantize"], batch=batch, capacity=cap)
    else:
        eng = make_engine(cfg, shape, batch, cap)
    if make_oracle is None:
        oracles = [O.OracleEngine(cfg, L, H, D, V, quantize=spec["quantize"], kv_heads=Hkv)
                   for _ in range(batch)]
    else:
        oracles = [make_oracle(cfg) for _ in range(batch)]
    pf = spec["prefill"]
    eng.begin_prefill(pf)
    kk = np.zeros((L, batch, pf, Hkv, D), np.float32)
    vv = np.zeros_like(kk)
    for b, orc in enumerate(oracles):
        orc.begin_prefill(pf)
        for layer in range(L):
            k, v = S.scenario_prefill_kv(spec, seq_seed(spec, b), layer)
            kk[layer, b], vv[layer, b] = k, v
            for pos in range(pf):
                orc.append_prefill(layer, k[pos], v[pos], pos)
    eng.prefill(torch.from_numpy(kk), torch.from_numpy(vv))

    worst_attn = 0.0
    gbuf = graph_obj = None
    mism = trials = 0
    for t in range(1, nsteps + 1):
        q = np.stack([np.stack([S.scenario_q(spec, seq_seed(spec, b), t, layer) for b in range(batch)])
                      for layer in range(L)])
        out, w = eng.attend_layers(torch.from_numpy(q), weights=True)
        out, w = out.cpu().numpy(), w.cpu().numpy()
        refs_all = [[orc.attend(layer, q[layer, b]) for layer in range(L)] for b, orc in enumerate(oracles)]
        if not use_gpu_rows:
            # the reference's trace-driver path: the caller supplies the rows (fp64)
            for layer in range(L):
                eng.stage_rows(layer, [refs_all[b][layer][1] for b in range(batch)])
        logits = np.stack([S.step_logits(seq_seed(spec, b), t, V) for b in range(batch)])
        kv = [[S.step_kv(seq_seed(spec, b), t, layer, Hkv, D) for b in range(batch)] for layer in range(L)]
        kn = np.stack([np.stack([kv[layer][b][0] for b in range(batch)]) for layer in range(L)])
        vn = np.stack([np.stack([kv[layer][b][1] for b in range(batch)]) for layer in range(L)])
        if production:
            staged_w = {(layer, b): eng.read_staged(layer, b, oracles[b].caches[layer].n)
                        for layer in range(L) for b in range(batch)}
            xs = dict(logits=torch.from_numpy(logits.astype(np.float32)), q=torch.from_numpy(q).half(),
                      k=torch.from_numpy(kn).half(), v=torch.from_numpy(vn).half())
            if graph and t >= 2:   # captured after one eager step, as the bench captures after warm-up
                if gbuf is None:
                    gbuf = {k: x.cuda() for k, x in xs.items()}
                    gout = torch.empty((L, batch, H, D), dtype=torch.float32, device="cuda")
                    graph_obj = eng.capture_step(gbuf["logits"], gbuf["k"], gbuf["v"], gbuf["q"], out=gout)
                for k, x in xs.items():
                    gbuf[k].copy_(x)
                graph_obj.replay()
                eng.note_replayed_steps(1)
                res_out = gout
                km_t, kl_t = eng._kept_map, eng._kept_len
            else:
                res = eng.step(xs["logits"], xs["k"], xs["v"], step=t, q=xs["q"])
                res_out, km_t, kl_t = res.out, res.kept_map, res.kept_len
            out_p = res_out.cpu().numpy()
            assert np.array_equal(out_p, out), f"{name} t={t}: production output != weights-dump output"
            for (layer, b), a in staged_w.items():
                ap = eng.read_staged(layer, b, a.size)
                assert np.array_equal(ap, a), f"{name} t={t} l={layer} b={b}: production head mean != dump path's"
            recs = eng.records()
            kept_map, kept_len = km_t.cpu().numpy(), kl_t.cpu().numpy()
        else:
            res = eng.step(torch.from_numpy(logits.astype(np.float32)), torch.from_numpy(kn),
                           torch.from_numpy(vn), step=t)
            recs = eng.records()
            kept_map = res.kept_map.cpu().numpy()
            kept_len = res.kept_len.cpu().numpy()
        if on_step is not None:
            on_step(t, recs)
        for b, orc in enumerate(oracles):
            rows, refs = [], []
            for layer in range(L):
                n = orc.caches[layer].n
                o_ref, w_ref = refs_all[b][layer]
                refs.append(o_ref)
                rows.append(w[layer, b, :, :n].astype(np.float64) if use_gpu_rows else w_ref)
            worst_attn = max(worst_attn, compare_attention(out[:, b], np.stack(refs), f"{name} t={t} b={b}"))
            if own_attention_trials:
                twin = copy.deepcopy(orc)
                _, kept_own = twin.step(logits[b], [refs_all[b][layer][1] for layer in range(L)],
                                        [(kn[l, b], vn[l, b]) for l in range(L)], t, return_kept=True)
                for layer in range(L):
                    m = kept_len[layer, b]
                    trials += 1
                    mism += int(not np.array_equal(kept_map[layer, b, :m], kept_own[layer]))
            rec, kept = orc.step(logits[b], rows, [(kn[l, b], vn[l, b]) for l in range(L)], t, return_kept=True)
            g = recs[b]
            for key in ("budget", "len_pre", "len_post", "evicted", "int8", "memory_bytes", "token"):
                assert getattr(g, key) == rec[key], f"{name} t={t} b={b} {key}: {getattr(g, key)} != {rec[key]}"
            for key in ("confidence", "entropy_norm", "margin", "margin_sig", "top_prob"):
                a, r = getattr(g, key), rec[key]
                assert abs(a - r) <= CONF_RTOL * max(1.0, abs(r)), f"{name} t={t} b={b} {key}: {a} vs {r}"
            for layer in range(L):
                m = kept_len[layer, b]
                assert np.array_equal(kept_map[layer, b, :m], kept[layer]), f"{name} t={t} b={b} l={layer} kept"
        if t % check_every == 0 or t == nsteps:
            for b, orc in enumerate(oracles):
                for layer in range(L):
                    compare_cache(eng.read_cache(layer, b), orc.caches[layer], f"{name} t={t} b={b} l={layer}")
    res = {"steps": nsteps, "worst_attn_rel": worst_attn, "kept_mismatch": mism, "kept_trials": trials}
    if spec.get("needle"):
        # run_decode's retention rule (simulator.py:464-467): the needle position is cached in
        # every layer (checked after the last step, on the GPU's own state)
        pos = spec["needle"]["pos"]
        res["needle_retained"] = [all(pos in eng.read_cache(layer, b)["positions"] for layer in range(L))
                                  for b in range(batch)]
    if on_end is not None:
        on_end(eng)
    eng.close()
    return res
