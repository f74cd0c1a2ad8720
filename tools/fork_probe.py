"""Probe: step time with K1 serial after K2 vs forked beside it (bench workload shapes)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402

quant = sys.argv[1] == "int8" if len(sys.argv) > 1 else True
L, H, Hkv, D, V, B, n = 32, 32, 8, 128, 128256, 8, 4096
cfg = PolicyConfig(n_high=4096, n_low=4096, protected_p=64, alpha=0.70, fp16_window_w=256, pyramid_n_min=96)
eng = ConfKVEngine(cfg, ModelShape(L, H, D, V, num_kv_heads=Hkv), quantize=quant, batch=B, capacity=n + 2)
g = torch.Generator(device="cuda").manual_seed(1)
eng.begin_prefill(n)
for layer in range(L):
    k = torch.randn((1, B, n, Hkv, D), generator=g, device="cuda").half()
    eng.prefill(k, torch.randn_like(k), layer_begin=layer)
x = dict(logits=(8 * torch.randn((B, V), generator=g, device="cuda")).float(),
         q=torch.randn((L, B, H, D), generator=g, device="cuda").half(),
         k=torch.randn((L, B, Hkv, D), generator=g, device="cuda").half(),
         v=torch.randn((L, B, Hkv, D), generator=g, device="cuda").half())
out = torch.empty((L, B, H, D), device="cuda")
t = 0
s = torch.cuda.current_stream()


def run(mode, steps):
    global t
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        t += 1
        if mode == "serial":
            ev[i][0].record(s)
            eng.attend_layers(x["q"], out=out)
            ev[i][1].record(s)
            eng.step(x["logits"], x["k"], x["v"], step=t, kept=False)
        elif mode == "attn_only":
            ev[i][0].record(s)
            eng.attend_layers(x["q"], out=out)
            ev[i][1].record(s)
        else:
            eng.step(x["logits"], x["k"], x["v"], step=t, q=x["q"], kept=False, out=out, attn_events=ev[i])
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3, sum(p.elapsed_time(q) for p, q in ev) / steps * 1e3


for rep in range(2):
    for mode in ("serial", "fork", "attn_only"):
        run(mode, 5)
        st, at = run(mode, 30)
        print(f"{'int8' if quant else 'fp16'} {mode:9s} step {st:7.1f} us  attention {at:7.1f} us", flush=True)
