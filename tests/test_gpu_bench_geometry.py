"""Parity at the benchmarked geometry itself (bench.py's default workload):
Llama-3-8B shape (L=32, Hq=32, Hkv=8, D=128, V=128,256), batch 8, a 4,096-entry bulk prefill,
N_high = N_low = 4,096, P=64, alpha=0.70, W=256, INT8 on (and the FP16 variant), steps replayed
from one `capture_step` CUDA graph exactly as bench.py times them.

At this size K2 runs the kernels the small scenarios never reach on their own:
k2_combine_staged<WD=false> (n4 * caches = 5 * 256 >= 4 * 148), the persistent tcgen05 grid
with its static-stride item schedule (256 caches * 8 heads * 9 splits >= 8 * 2 * 148 items) and
the general kernel in unit mode. Per step:
  1. attention with the weights dump (WD=true) -> the weights the oracle consumes;
  2. the production graph replay (attention WD=false + K1 + K3/K4 + kept map);
  3. production output == dump output bit for bit (all 256 caches), production staged head
     mean == dump path's bit for bit (sampled caches), and for sampled (layer, sequence)
     caches an oracle (pinned to the reference) fed the dumped weights must agree exactly on
     kept sets, records, EMA, positions, INT8 codes and scales; the oracle's own fp64
     attention must match the GPU output within 1e-3.
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
from tests.gpu_driver import CONF_RTOL, compare_attention, compare_cache  # noqa: E402

L, H, HKV, D, V, B, N = 32, 32, 8, 128, 128256, 8, 4096
SAMPLES = [(0, 0), (9, 3), (17, 7), (31, 5)]    # (layer, sequence) caches checked against the oracle
STEPS = 5


@pytest.mark.parametrize("quantize", [True, False], ids=["int8", "fp16"])
def test_bench_geometry_production_graph(quantize):
    cfg = PolicyConfig(n_high=N, n_low=N, protected_p=64, alpha=0.70, fp16_window_w=256, pyramid_n_min=96)
    shape = ModelShape(L, H, D, V, num_kv_heads=HKV)
    dev = torch.device("cuda", 0)
    eng = ConfKVEngine(cfg, shape, quantize=quantize, batch=B, capacity=N + 2, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    eng.begin_prefill(N)
    oracles = {}
    for layer in range(L):
        k = torch.randn((1, B, N, HKV, D), generator=g, device=dev).half()
        v = torch.randn((1, B, N, HKV, D), generator=g, device=dev).half()
        eng.prefill(k, v, layer_begin=layer)
        for (sl, sb) in SAMPLES:
            if sl == layer:
                orc = O.OracleEngine(cfg, 1, H, D, V, quantize=quantize, kv_heads=HKV)
                orc.begin_prefill(N)
                orc.caches[0].bulk_append(k[0, sb].float().cpu().numpy(), v[0, sb].float().cpu().numpy(), 0, -N)
                oracles[(sl, sb)] = orc
    del k, v
    buf = dict(logits=torch.empty((B, V), device=dev), q=torch.empty((L, B, H, D), device=dev, dtype=torch.half),
               k=torch.empty((L, B, HKV, D), device=dev, dtype=torch.half),
               v=torch.empty((L, B, HKV, D), device=dev, dtype=torch.half))
    out_g = torch.empty((L, B, H, D), dtype=torch.float32, device=dev)
    graph = None
    worst = 0.0
    for t in range(1, STEPS + 1):
        gain = torch.where(torch.rand((B, 1), generator=g, device=dev) < 0.75, 8.0, 0.5)
        buf["logits"].copy_(gain * torch.randn((B, V), generator=g, device=dev))
        buf["q"].copy_(torch.randn((L, B, H, D), generator=g, device=dev))
        buf["k"].copy_(torch.randn((L, B, HKV, D), generator=g, device=dev))
        buf["v"].copy_(torch.randn((L, B, HKV, D), generator=g, device=dev))
        n_pre = {s: o.caches[0].n for s, o in oracles.items()}
        # 1. weights-dumping attention: the rows the oracle consumes
        out_w, w = eng.attend_layers(buf["q"], weights=True)
        staged = {s: eng.read_staged(s[0], s[1], n_pre[s]) for s in oracles}
        rows = {s: w[s[0], s[1], :, : n_pre[s]].double().cpu().numpy() for s in oracles}
        out_w = out_w.cpu().numpy()
        del w
        # 2. the production step: eager at step 1 (bulk demotion), then one captured graph
        if t == 1:
            res = eng.step(buf["logits"], buf["k"], buf["v"], step=t, q=buf["q"], out=out_g)
        else:
            if graph is None:
                graph = eng.capture_step(buf["logits"], buf["k"], buf["v"], buf["q"], out=out_g)
            graph.replay()
            eng.note_replayed_steps(1)
        recs = eng.records()
        out_p = out_g.cpu().numpy()
        kept_map, kept_len = eng._kept_map.cpu().numpy(), eng._kept_len.cpu().numpy()
        # 3. production == dump path, bit for bit
        assert np.array_equal(out_p, out_w), f"t={t}: production output differs from the dump path's"
        for s, a in staged.items():
            assert np.array_equal(eng.read_staged(s[0], s[1], a.size), a), f"t={t} {s}: staged head mean differs"
        logits = buf["logits"].double().cpu().numpy()
        q = buf["q"].float().cpu().numpy()
        kn, vn = buf["k"].float().cpu().numpy(), buf["v"].float().cpu().numpy()
        for (sl, sb), orc in oracles.items():
            o_ref, _ = orc.attend(0, q[sl, sb])
            worst = max(worst, compare_attention(out_p[sl, sb][None], o_ref[None], f"t={t} l={sl} b={sb}"))
            rec, kept = orc.step(logits[sb], [rows[(sl, sb)]], [(kn[sl, sb], vn[sl, sb])], t, return_kept=True)
            gr = recs[sb]
            assert gr.budget == rec["budget"] and gr.token == rec["token"], (t, sl, sb)
            for key in ("len_pre", "len_post", "evicted", "int8"):
                assert getattr(gr, key)[sl] == rec[key][0], (t, sl, sb, key, getattr(gr, key)[sl], rec[key][0])
            for key in ("confidence", "entropy_norm", "margin", "margin_sig", "top_prob"):
                assert abs(getattr(gr, key) - rec[key]) <= CONF_RTOL * max(1.0, abs(rec[key])), (t, key)
            m = kept_len[sl, sb]
            assert np.array_equal(kept_map[sl, sb, :m], kept[0]), f"t={t} l={sl} b={sb}: kept set"
    for (sl, sb), orc in oracles.items():
        compare_cache(eng.read_cache(sl, sb), orc.caches[0], f"final l={sl} b={sb}")
    assert worst < 1e-3
    eng.close()
