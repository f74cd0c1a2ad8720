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
for t in range(1, 61):
    loop.step()
    torch.cuda.synchronize()
    bad = ~torch.isfinite(loop.attn)
    if bad.any():
        idx = bad.nonzero()[:5].tolist()
        print("step", t, "non-finite attn at", idx, "count", int(bad.sum()))
        for l in range(4):
            for b in range(B):
                c = eng.read_cache(l, b)
                print(" l", l, "b", b, "n", c["valid_len"], "nseg", c["num_segments"], "segs", np.unique(c["segment_of"])[:10], "int8", int((c["segment_of"]>=0).sum()))
        rec = eng._rec_l
        print([ (r.len_after, r.int8_count, r.int8_codes) for r in rec][:12])
        break
    if not torch.isfinite(loop.logits).all():
        print("logits nonfinite at", t); break
else:
    print("no nan")

# replay layer 0 attention with weights for the failing step's q
q = loop.q[0:1].clone()
out, w = eng.attend_layers(q, 0, weights=True)
torch.cuda.synchronize()
w = w[0, 0].cpu().numpy()   # [Hq, cap]
c = eng.read_cache(0, 0)
n = c["valid_len"]
badh = np.where(~np.isfinite(w[:, :n]).all(axis=1) | np.isnan(w[:, :n]).any(axis=1))[0]
print("heads with nan weights", badh)
for h in badh[:2]:
    be = np.where(~np.isfinite(w[h, :n]))[0]
    print(" head", h, "bad entries", be[:20], "segs", c["segment_of"][be[:20]])
print("q finite", bool(torch.isfinite(q).all()), "q absmax", float(q.abs().max()))
print("keys absmax", float(np.abs(c["keys"][:n]).max()), "vals absmax", float(np.abs(c["values"][:n]).max()))
print("seg scales k min/max", c["seg_k_scale"].min(), c["seg_k_scale"].max(), "counts", c["seg_count"])
