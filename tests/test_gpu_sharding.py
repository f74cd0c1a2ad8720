"""Head sharding and vocab sharding on one GPU with W logical shards: W
engines each own Hkv/W KV heads; the all-gather is a device-side stack (what
parallel.HeadShardedStep does over NCCL). Every shard must reproduce the unsharded
engine bit-for-bit: kept maps, records, EMA, INT8 codes/scales of its heads, outputs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import confkv_oracle as O  # noqa: E402
from oracle import scenarios as S  # noqa: E402
from paper_2605_24786_b200.config import ModelShape, PolicyConfig  # noqa: E402
from paper_2605_24786_b200.engine import ConfKVEngine  # noqa: E402


@pytest.mark.parametrize("W,Hq,Hkv,D,exchange", [
    (2, 8, 4, 64, "chain"), (4, 8, 4, 64, "chain"), (2, 8, 4, 64, "gather"),
    # C3's 8-GPU layout: Qwen-32B heads (40 query / 8 KV, group 5), one KV head per rank
    (8, 40, 8, 128, "chain"), (8, 40, 8, 128, "gather")])
def test_head_sharded_equals_unsharded(W, Hq, Hkv, D, exchange):
    L, V, B, pf, steps = 2, 500, 2, 70, 45
    cfg = PolicyConfig(n_high=40, n_low=64, protected_p=8, pyramid_n_min=24, fp16_window_w=16, alpha=0.7)
    cap = 80
    full = ConfKVEngine(cfg, ModelShape(L, Hq, D, V, num_kv_heads=Hkv), quantize=True, batch=B, capacity=cap)
    hq, hk = Hq // W, Hkv // W
    shards = [ConfKVEngine(cfg, ModelShape(L, hq, D, V, num_kv_heads=hk), quantize=True, batch=B, capacity=cap)
              for _ in range(W)]
    g = torch.Generator().manual_seed(3)
    k = torch.randn((L, B, pf, Hkv, D), generator=g).half()
    v = torch.randn((L, B, pf, Hkv, D), generator=g).half()
    full.begin_prefill(pf)
    full.prefill(k, v)
    for r, e in enumerate(shards):
        e.begin_prefill(pf)
        e.prefill(k[:, :, :, r * hk:(r + 1) * hk].contiguous(), v[:, :, :, r * hk:(r + 1) * hk].contiguous())
    for t in range(1, steps + 1):
        q = torch.randn((L, B, Hq, D), generator=g).half().cuda()
        kn = torch.randn((L, B, Hkv, D), generator=g).half().cuda()
        vn = torch.randn((L, B, Hkv, D), generator=g).half().cuda()
        logits = torch.tensor(np.stack([S.step_logits(9 + b, t, V) for b in range(B)]), dtype=torch.float32).cuda()
        res = full.step(logits, kn, vn, step=t, q=q)
        ref_recs = full.records()
        outs, ws = [], []
        for r, e in enumerate(shards):
            o, w = e.attend_layers(q[:, :, r * hq:(r + 1) * hq].contiguous(), weights=True)
            outs.append(o)
            ws.append(w)
        if exchange == "chain":
            # parallel.chain_head_sums over W ranks, in process: rank r adds its heads to rank
            # r-1's fp64 running sums; every rank stages the last rank's sums / Hq
            acc = torch.empty((L, B, cap), dtype=torch.float64, device="cuda")
            for r, e in enumerate(shards):
                e.head_partial(ws[r], acc if r else None, acc)
            for e in shards:
                e.stage_mass(acc, Hq)
        else:
            gathered = torch.stack(ws)
            for e in shards:
                e.stage_weights(gathered, W)
        shard_res = []
        for r, e in enumerate(shards):
            e.confidence(logits)
            shard_res.append(e.manage(kn[:, :, r * hk:(r + 1) * hk].contiguous(), vn[:, :, r * hk:(r + 1) * hk].contiguous(), t))
        assert torch.equal(torch.cat(outs, dim=2), res.out), f"t={t}: outputs"
        recs = [e.records() for e in shards]
        for b in range(B):
            mem = 0
            for r in range(W):
                a, f = recs[r][b], ref_recs[b]
                for key in ("budget", "len_pre", "len_post", "evicted", "int8", "token", "confidence"):
                    assert getattr(a, key) == getattr(f, key), (t, r, b, key)
                mem += a.memory_bytes
            assert mem == ref_recs[b].memory_bytes
        for r in range(W):
            kl = res.kept_len
            assert torch.equal(shard_res[r].kept_len, kl)
            for l in range(L):
                for b in range(B):
                    m = int(kl[l, b])
                    assert torch.equal(shard_res[r].kept_map[l, b, :m], res.kept_map[l, b, :m])
        if t % 15 == 0:
            for l in range(L):
                for b in range(B):
                    fc = full.read_cache(l, b)
                    for r, e in enumerate(shards):
                        sc = e.read_cache(l, b)
                        sl = slice(r * hk, (r + 1) * hk)
                        assert np.array_equal(sc["ema"], fc["ema"])
                        assert np.array_equal(sc["positions"], fc["positions"])
                        assert np.array_equal(sc["segment_of"], fc["segment_of"])
                        assert np.array_equal(sc["k_codes"], fc["k_codes"][:, sl])
                        assert np.array_equal(sc["v_codes"], fc["v_codes"][:, sl])
                        assert np.array_equal(sc["seg_k_scale"], fc["seg_k_scale"][:, sl])
                        assert np.array_equal(sc["keys"], fc["keys"][:, sl])


@pytest.mark.parametrize("W", [2, 3, 8])
def test_vocab_sharded_confidence(W):
    V, B = 128256, 4
    rows = [S.step_logits(41, t, V) for t in range(1, B + 1)]
    logits = torch.tensor(np.stack(rows), dtype=torch.float32).cuda()
    bounds = [(r * V) // W for r in range(W + 1)]
    cfg = PolicyConfig()
    engines = [ConfKVEngine(cfg, ModelShape(1, 1, 16, bounds[r + 1] - bounds[r]), batch=B, capacity=300)
               for r in range(W)]
    parts = torch.stack([e.confidence_partial(logits[:, bounds[r]:bounds[r + 1]].contiguous(), bounds[r])
                         for r, e in enumerate(engines)])
    engines[0].confidence_merge(parts, V)
    recs = engines[0].records()
    for b in range(B):
        f = O.confidence(O.softmax64(rows[b]))
        g = recs[b]
        for key in ("entropy_norm", "margin", "margin_sig", "top_prob"):
            assert abs(getattr(g, key) - f[key]) <= 1e-9 * max(1.0, abs(f[key])), (W, b, key)
        assert abs(g.confidence - f["score"]) <= 1e-12
        assert g.token == int(np.argmax(rows[b]))
        assert g.budget == O.select_tier(f["score"], cfg.n_high, cfg.n_low, cfg.tau)
