import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2605_24786_b200.config import ModelShape, PolicyConfig
from paper_2605_24786_b200.engine import ConfKVEngine
from paper_2605_24786_b200.decode import DecodeLoop, DecodeModel
shape = ModelShape(num_layers=4, num_heads=8, head_dim=128, vocab_size=3000, num_kv_heads=2)
cfg = PolicyConfig(n_high=96, n_low=160, protected_p=16, pyramid_n_min=96, fp16_window_w=32, alpha=0.7)
B, P = 3, 40
prompt = torch.randint(0, shape.vocab_size, (B, P), generator=torch.Generator().manual_seed(2))
eng = ConfKVEngine(cfg, shape, quantize=True, batch=B, capacity=200)
model = DecodeModel(shape, seed=9, dtype=torch.bfloat16)
loop = DecodeLoop(eng, model, use_graph=False)
loop.prefill(prompt)
orig = eng.attend_layers
state = {"t": 0, "done": False}
def patched(q, layer_begin=0, stream=None, weights=False, out=None):
    r = orig(q, layer_begin, stream, weights, out)
    torch.cuda.synchronize()
    o = r[0]
    if not state["done"] and not torch.isfinite(o).all():
        state["done"] = True
        print("NaN at step", state["t"], "layer", layer_begin, flush=True)
        for rep in range(3):
            o2, w2 = orig(q.clone(), layer_begin, None, True, None)
            torch.cuda.synchronize()
            print(" rerun", rep, "finite", bool(torch.isfinite(o2).all()), "w finite", bool(torch.isfinite(w2).all()))
        o2, w2 = orig(q.clone(), layer_begin, None, True, None)
        w2 = w2[0].cpu().numpy()
        for b in range(B):
            c = eng.read_cache(layer_begin, b)
            n = c["valid_len"]
            bad = ~np.isfinite(w2[b, :, :n])
            if bad.any():
                hs, es = np.nonzero(bad)
                print(" b", b, "bad heads", np.unique(hs), "entries", np.unique(es)[:20], "n", n, "segs", c["segment_of"][np.unique(es)[:20]])
                print("  q absmax", float(q[0, b].abs().max()), "scales", c["seg_k_scale"].min(), c["seg_count"])
    return r
eng.attend_layers = patched
for t in range(1, 61):
    state["t"] = t
    loop.step()
    if state["done"]:
        break
print("end")
