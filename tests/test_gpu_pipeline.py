"""HostPipeline (host-buffer, copy-overlapped steps) must give exactly what the device-resident
ConfKVEngine.step gives on the same inputs: attention outputs bit for bit, identical records,
identical kept-index maps (the pipeline carries them in compact victim-list form)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine, HostPipeline  # noqa: E402


@pytest.mark.parametrize("depth,graphs,packed,fused", [
    (1, False, False, False), (2, False, False, False), (3, False, False, False),
    (1, True, False, False), (2, True, False, False), (3, True, False, False),
    (2, False, True, False),
    (2, True, True, False),    # steady state through ckv_pipe_submit (one C call per step)
    (3, True, True, False),
    (2, True, True, True)])    # H2D / D2H captured into each set's graph (fused copies)
def test_pipeline_matches_device_steps(depth, graphs, packed, fused):
    L, Hq, Hkv, D, V, B, pf, steps = 2, 8, 2, 128, 1000, 3, 300, 40
    cfg = PolicyConfig(n_high=200, n_low=280, protected_p=16, pyramid_n_min=96, fp16_window_w=32, alpha=0.7)
    shape = ModelShape(L, Hq, D, V, num_kv_heads=Hkv)
    engines = [ConfKVEngine(cfg, shape, quantize=True, batch=B, capacity=320) for _ in range(2)]
    g = torch.Generator().manual_seed(11)
    k = torch.randn((L, B, pf, Hkv, D), generator=g).half()
    v = torch.randn((L, B, pf, Hkv, D), generator=g).half()
    for e in engines:
        e.begin_prefill(pf)
        e.prefill(k.cuda(), v.cuda())
    ins = []
    for t in range(1, steps + 1):
        ins.append(dict(logits=(torch.randn((B, V), generator=g) * (8.0 if t % 4 else 0.5)).float(),
                        q=torch.randn((L, B, Hq, D), generator=g).half(),
                        k=torch.randn((L, B, Hkv, D), generator=g).half(),
                        v=torch.randn((L, B, Hkv, D), generator=g).half()))
    ref_out, ref_rec, ref_kept = [], [], []
    for t, x in enumerate(ins, 1):
        r = engines[0].step(x["logits"].cuda(), x["k"].cuda(), x["v"].cuda(), step=t, q=x["q"].cuda())
        ref_out.append(r.out.cpu())
        ref_rec.append(engines[0].records())
        km, kl = r.kept_map.cpu().numpy(), r.kept_len.cpu().numpy()
        ref_kept.append([[km[layer, b, :kl[layer, b]] for b in range(B)] for layer in range(L)])
    pipe = HostPipeline(engines[1], depth=depth, graphs=graphs, fused_copies=fused)
    # packed: host_inputs() buffers, one per input set (with graphs and small steps the
    # pipeline then captures the H2D / D2H copies into each set's graph: fused_copies)
    sets = [pipe.host_inputs() for _ in range(depth)] if packed else None
    pins = [{kk: vv.pin_memory() for kk, vv in x.items()} for x in ins]
    outs = [torch.empty_like(ref_out[0]).pin_memory() for _ in range(depth)]
    assert pipe.fused == (fused and graphs)
    for t, x in enumerate(pins, 1):
        if packed:   # safe to refill: the previous user of this set was drained below
            for kk, vv in x.items():
                sets[t % depth][kk].copy_(vv)
            x = sets[t % depth]
        pipe.submit(t, x["logits"], x["q"], x["k"], x["v"], out=outs[t % depth])
        if t > 1 and depth > 1:
            assert pipe.records(t - 1) == ref_rec[t - 2], f"step {t - 1}: records (one step behind)"
        pipe.records(t)
        torch.cuda.current_stream().wait_stream(pipe.d2h)
        pipe.drain()
        assert torch.equal(outs[t % depth], ref_out[t - 1]), f"step {t}: output"
        assert pipe.records(t) == ref_rec[t - 1], f"step {t}: records"
        kept = pipe.kept(t)
        for layer in range(L):
            for b in range(B):
                assert np.array_equal(kept[layer][b], ref_kept[t - 1][layer][b]), f"step {t}: kept map"
    if graphs and packed and not fused:
        assert pipe.c_submits >= len(pins) - 2 * depth, "steady state did not go through ckv_pipe_submit"


@pytest.mark.parametrize("quantize", [False, True])
def test_fused_step_paths_agree(quantize):
    """Three ways to run a step must agree bit for bit: separate attend + step calls (serial),
    ConfKVEngine.step(q=...) (K1 forked onto a torch side stream) and the C ABI ckv_step
    (K1 forked onto the engine-owned side stream inside the library), FP16 and INT8 (persistent
    tcgen05 K2) caches."""
    import ctypes as C

    from paper_2605_24786_b200 import _lib
    L, Hq, Hkv, D, V, B, pf, steps = 3, 8, 2, 128, 70000, 2, 600, 24
    cfg = PolicyConfig(n_high=520, n_low=600, protected_p=16, pyramid_n_min=96, fp16_window_w=64, alpha=0.7)
    shape = ModelShape(L, Hq, D, V, num_kv_heads=Hkv)
    engines = [ConfKVEngine(cfg, shape, quantize=quantize, batch=B, capacity=640) for _ in range(3)]
    g = torch.Generator().manual_seed(5)
    k = torch.randn((L, B, pf, Hkv, D), generator=g).half().cuda()
    v = torch.randn((L, B, pf, Hkv, D), generator=g).half().cuda()
    for e in engines:
        e.begin_prefill(pf)
        e.prefill(k, v)
    for t in range(1, steps + 1):
        x = dict(logits=(torch.randn((B, V), generator=g) * (8.0 if t % 3 else 0.5)).float().cuda(),
                 q=torch.randn((L, B, Hq, D), generator=g).half().cuda(),
                 k=torch.randn((L, B, Hkv, D), generator=g).half().cuda(),
                 v=torch.randn((L, B, Hkv, D), generator=g).half().cuda())
        o0, _ = engines[0].attend_layers(x["q"])
        engines[0].step(x["logits"], x["k"], x["v"], step=t)
        o1 = engines[1].step(x["logits"], x["k"], x["v"], step=t, q=x["q"]).out
        e2 = engines[2]
        o2 = torch.empty_like(o0)
        _lib.check(e2.lib.ckv_step(e2._h, t, C.c_void_p(x["logits"].data_ptr()), _lib.DTYPE_F32, V,
                                   C.c_void_p(x["q"].data_ptr()), C.c_void_p(x["k"].data_ptr()),
                                   C.c_void_p(x["v"].data_ptr()), C.c_void_p(o2.data_ptr()),
                                   C.c_void_p(e2._kept_map.data_ptr()), C.c_void_p(e2._kept_len.data_ptr()),
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        e2._last_step = t
        torch.cuda.synchronize()
        assert torch.equal(o0, o1) and torch.equal(o0, o2), f"step {t}: attention outputs differ"
        r0, r1, r2 = engines[0].records(), engines[1].records(), engines[2].records()
        assert r0 == r1 == r2, f"step {t}: records differ"
        kl = engines[0]._kept_len.cpu()
        assert torch.equal(kl, engines[1]._kept_len.cpu()) and torch.equal(kl, engines[2]._kept_len.cpu())
        km = [e._kept_map.cpu() for e in engines]
        for li in range(L):
            for b in range(B):
                n = int(kl[li, b])
                assert torch.equal(km[0][li, b, :n], km[1][li, b, :n]), f"step {t}: kept map"
                assert torch.equal(km[0][li, b, :n], km[2][li, b, :n]), f"step {t}: kept map (ckv_step)"


@pytest.mark.parametrize("quantize", [False, True])
def test_captured_steps_match_eager(quantize):
    """ConfKVEngine.capture_step: K graphs captured in a row and replayed in order give the same
    outputs, records and caches as K eager steps (the step counter advances on the device)."""
    L, Hq, Hkv, D, V, B, pf, K = 2, 8, 2, 128, 3000, 2, 700, 12
    cfg = PolicyConfig(n_high=600, n_low=700, protected_p=16, pyramid_n_min=96, fp16_window_w=64, alpha=0.7)
    shape = ModelShape(L, Hq, D, V, num_kv_heads=Hkv)
    engines = [ConfKVEngine(cfg, shape, quantize=quantize, batch=B, capacity=720) for _ in range(2)]
    g = torch.Generator().manual_seed(3)
    k = torch.randn((L, B, pf, Hkv, D), generator=g).half().cuda()
    for e in engines:
        e.begin_prefill(pf)
        e.prefill(k, k)
    pool = [dict(logits=(torch.randn((B, V), generator=g) * s).float().cuda(),
                 q=torch.randn((L, B, Hq, D), generator=g).half().cuda(),
                 k=torch.randn((L, B, Hkv, D), generator=g).half().cuda(),
                 v=torch.randn((L, B, Hkv, D), generator=g).half().cuda()) for s in (8.0, 0.5)]
    for t in range(1, 3):   # two eager steps first on both
        for e in engines:
            x = pool[t % 2]
            e.step(x["logits"], x["k"], x["v"], step=t, q=x["q"])
    outs = [torch.empty((L, B, Hq, D), device="cuda") for _ in range(K)]
    graphs = [engines[1].capture_step(pool[(3 + i) % 2]["logits"], pool[(3 + i) % 2]["k"], pool[(3 + i) % 2]["v"],
                                      pool[(3 + i) % 2]["q"], out=outs[i]) for i in range(K)]
    ref_out, ref_rec = [], []
    for i in range(K):
        x = pool[(3 + i) % 2]
        ref_out.append(engines[0].step(x["logits"], x["k"], x["v"], step=3 + i, q=x["q"]).out.clone())
        ref_rec.append(engines[0].records())
    for i in range(K):
        graphs[i].replay()
        engines[1].note_replayed_steps(1)
        torch.cuda.synchronize()
        assert torch.equal(outs[i], ref_out[i]), i
        assert engines[1].records() == ref_rec[i], i
    for layer in range(L):
        for b in range(B):
            a, c = engines[0].read_cache(layer, b), engines[1].read_cache(layer, b)
            for key in ("positions", "steps", "ema", "segment_of", "k_codes"):
                assert np.array_equal(a[key], c[key]), key
    # an eager step after the replays continues from the device's step counter
    x = pool[(3 + K) % 2]
    for e in engines:
        e.step(x["logits"], x["k"], x["v"], step=3 + K, q=x["q"])
    assert engines[0].records() == engines[1].records()
