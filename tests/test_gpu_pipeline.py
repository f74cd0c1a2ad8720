"""HostPipeline (host-buffer, copy-overlapped steps) must give exactly what the device-resident
ConfKVEngine.step gives on the same inputs: attention outputs bit for bit, identical records."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine, HostPipeline  # noqa: E402


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_pipeline_matches_device_steps(depth):
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
    ref_out, ref_rec = [], []
    for t, x in enumerate(ins, 1):
        r = engines[0].step(x["logits"].cuda(), x["k"].cuda(), x["v"].cuda(), step=t, q=x["q"].cuda(), kept=False)
        ref_out.append(r.out.cpu())
        ref_rec.append(engines[0].records())
    pipe = HostPipeline(engines[1], depth=depth)
    pins = [{kk: vv.pin_memory() for kk, vv in x.items()} for x in ins]
    outs = [torch.empty_like(ref_out[0]).pin_memory() for _ in range(depth)]
    for t, x in enumerate(pins, 1):
        pipe.submit(t, x["logits"], x["q"], x["k"], x["v"], out=outs[t % depth])
        if t > 1 and depth > 1:
            assert pipe.records(t - 1) == ref_rec[t - 2], f"step {t - 1}: records (one step behind)"
        pipe.records(t)
        torch.cuda.current_stream().wait_stream(pipe.d2h)
        pipe.drain()
        assert torch.equal(outs[t % depth], ref_out[t - 1]), f"step {t}: output"
        assert pipe.records(t) == ref_rec[t - 1], f"step {t}: records"
