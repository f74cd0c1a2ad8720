"""F1: the decode loop (DecodeModel + ConfKVEngine, graph-replayed) against the fp64
restatement of ReferenceModel.forward (oracle.reference_forward, simulator.py:58-92)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import confkv_oracle as O  # noqa: E402
from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.decode import DecodeLoop, DecodeModel, run_decode  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402

LOGIT_RTOL = 1e-3


def _weights(shape, seed):
    L, Hq, Hkv, D, V = shape.num_layers, shape.num_heads, shape.kv_heads, shape.head_dim, shape.vocab_size
    d = Hq * D
    g = torch.Generator().manual_seed(seed)
    s = 1.0 / np.sqrt(d)
    r = lambda *sz, k=1.0: (torch.randn(sz, generator=g, dtype=torch.float64) * k).float()  # noqa: E731
    return dict(embedding=r(V, d), w_q=r(L, d, d, k=s), w_k=r(L, d, Hkv * D, k=s), w_v=r(L, d, Hkv * D, k=s),
                w_o=r(L, d, d, k=s), w_out=r(d, V, k=8.0 * s))


@pytest.mark.parametrize("kv_heads,quantize", [(4, False), (2, False), (2, True)])
def test_decode_forward_matches_reference(kv_heads, quantize):
    torch.backends.cuda.matmul.allow_tf32 = False
    shape = ModelShape(num_layers=3, num_heads=4, head_dim=64, vocab_size=700, num_kv_heads=kv_heads)
    cfg = PolicyConfig(n_high=24, n_low=40, protected_p=8, pyramid_n_min=16, fp16_window_w=8, alpha=0.65)
    B, P, steps = 2, 12, 40
    eng = ConfKVEngine(cfg, shape, quantize=quantize, batch=B, capacity=64)
    w = _weights(shape, 3)
    model = DecodeModel(shape, dtype=torch.float32, weights=w)
    wn = {k: v.double().numpy() for k, v in w.items()}
    loop = DecodeLoop(eng, model, use_graph=False)
    prompt = torch.randint(0, shape.vocab_size, (B, P), generator=torch.Generator().manual_seed(1))
    loop.prefill(prompt)
    tokens = prompt[:, -1].numpy().copy()
    worst = 0.0
    for t in range(1, steps + 1):
        pre = [[eng.read_cache(layer, b) for layer in range(shape.num_layers)] for b in range(B)]
        loop.step()
        recs = loop.records()
        lg = loop.logits.cpu().double().numpy()
        for b in range(B):
            kv = [(c["keys"], c["values"]) for c in pre[b]]
            ref, _, new_kv = O.reference_forward(tokens[b], kv, wn, shape.num_heads, shape.head_dim,
                                                 q_dtype=np.float16)   # the engine's q input type
            err = np.abs(lg[b] - ref).max() / np.abs(ref).max()
            worst = max(worst, err)
            assert err <= LOGIT_RTOL, f"step {t} seq {b}: logits rel err {err:.2e}"
            assert recs[b].token == int(np.argmax(lg[b])), f"step {t} seq {b}: greedy token"
            # the appended entry is this step's K/V (fp16-rounded) at the step's position
            post = eng.read_cache(0, b)
            assert post["positions"][-1] == P + t - 1 and post["steps"][-1] == t
            kref = new_kv[0][0].astype(np.float16).astype(np.float32)
            assert np.abs(post["keys"][-1] - kref).max() <= 2e-3 * np.abs(kref).max()
            tokens[b] = recs[b].token
    assert worst < LOGIT_RTOL


def test_graph_replay_equals_eager():
    """The graph-captured loop gives the same tokens, records and caches as the eager loop."""
    shape = ModelShape(num_layers=4, num_heads=8, head_dim=128, vocab_size=3000, num_kv_heads=2)
    cfg = PolicyConfig(n_high=96, n_low=160, protected_p=16, pyramid_n_min=96, fp16_window_w=32, alpha=0.7)
    B, P, steps = 3, 40, 60
    prompt = torch.randint(0, shape.vocab_size, (B, P), generator=torch.Generator().manual_seed(2))
    runs = []
    for use_graph in (False, True):
        eng = ConfKVEngine(cfg, shape, quantize=True, batch=B, capacity=200)
        model = DecodeModel(shape, seed=9, dtype=torch.bfloat16)
        recs = run_decode(eng, model, prompt, steps, use_graph=use_graph)
        caches = [eng.read_cache(layer, b) for layer in range(shape.num_layers) for b in range(B)]
        runs.append((recs, caches))
    (r0, c0), (r1, c1) = runs
    assert r0 == r1
    for a, b in zip(c0, c1):
        for k in ("positions", "steps", "ema", "segment_of", "keys", "values", "k_codes", "v_codes"):
            assert np.array_equal(a[k], b[k]), k
    # the decode actually exercised the policy: evictions and INT8 demotions happened
    assert any(sum(r.evicted) for step in r0 for r in step)
    assert any(sum(r.int8) for step in r0 for r in step)
