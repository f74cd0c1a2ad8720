"""Probe: per-op device time of one decode-loop layer at Llama-8B shape, batch 8, 4K INT8."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.decode import DecodeLoop, DecodeModel  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402

quant = (sys.argv[1] if len(sys.argv) > 1 else "int8") == "int8"
L, H, Hkv, D, V, B, n = 32, 32, 8, 128, 128256, 8, 4096
cfg = PolicyConfig(n_high=4096, n_low=4096, protected_p=64, alpha=0.70, fp16_window_w=256, pyramid_n_min=96)
shape = ModelShape(L, H, D, V, num_kv_heads=Hkv)
eng = ConfKVEngine(cfg, shape, quantize=quant, batch=B, capacity=n + 2)
g = torch.Generator(device="cuda").manual_seed(1)
eng.begin_prefill(n)
for layer in range(L):
    k = torch.randn((1, B, n, Hkv, D), generator=g, device="cuda").half()
    eng.prefill(k, torch.randn_like(k), layer_begin=layer)
model = DecodeModel(shape, seed=3)
loop = DecodeLoop(eng, model)
for _ in range(4):
    loop.step()
torch.cuda.synchronize()
x = torch.randn(B, H * D, device="cuda")
xb = x.bfloat16()
o = torch.randn(B, H * D, device="cuda").bfloat16()
q = torch.randn(1, B, H, D, device="cuda").half()
out = torch.empty(1, B, H, D, device="cuda")


def tm(name, f, it=50):
    for _ in range(5):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        f()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / it * 1e3:8.1f} us", flush=True)


tm("qkv gemm", lambda: torch.matmul(xb, model.w_qkv[3]))
tm("o gemm addmm", lambda: torch.addmm(x, o, model.w_o[3], out_dtype=torch.float32))
tm("out gemm", lambda: torch.mm(xb, model.w_out, out_dtype=torch.float32))
tm("attend 1 layer", lambda: eng.attend_layers(q, 3, out=out))
tm("attend 32 layers", lambda: eng.attend_layers(loop.q, 0, out=loop.attn), it=10)
tm("decode step (graph)", loop.step, it=20)
