"""Phase timing of K3 (manage) from a -DCKV_TRACE build (debug tool, GPU box).

  CKV_NVCC_EXTRA=-DCKV_TRACE python -m paper_2605_24786_b200.build --force
  python tools/trace_k3.py [--workload llama8b_int8_4k]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
NAMES = ["prologue", "EMA commit", "rank+select", "compaction", "INT8 window", "append"]


def main():
    import torch
    import bench
    from paper_2605_24786_b200.config import ModelShape, PolicyConfig
    from paper_2605_24786_b200.engine import ConfKVEngine
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama8b_int8_4k")
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda", 0)
    L, H, Hkv, D, V, B, n = wl["L"], wl["H"], wl["Hkv"], wl["D"], wl["V"], wl["B"], wl["n"]
    cfg = PolicyConfig(**wl["cfg"])
    eng = ConfKVEngine(cfg, ModelShape(L, H, D, V, num_kv_heads=Hkv), quantize=wl["quantize"], batch=B,
                       capacity=max(n, cfg.n_low) + 2, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    eng.begin_prefill(n)
    for layer in range(L):
        k = torch.randn((1, B, n, Hkv, D), generator=g, device=dev).half()
        eng.prefill(k, torch.randn_like(k), layer_begin=layer)
    x = dict(logits=(8 * torch.randn((B, V), generator=g, device=dev)).float(),
             q=torch.randn((L, B, H, D), generator=g, device=dev).half(),
             k=torch.randn((L, B, Hkv, D), generator=g, device=dev).half(),
             v=torch.randn((L, B, Hkv, D), generator=g, device=dev).half())
    for t in range(1, 6):
        eng.step(x["logits"], x["k"], x["v"], step=t, q=x["q"], kept=False)
    torch.cuda.synchronize()
    C_ = L * B
    buf = np.zeros((4096, 8), np.uint64)
    eng.lib.ckv_debug_k3trace.restype = C.c_int
    eng.lib.ckv_debug_k3trace(C.c_void_p(buf.ctypes.data), C.c_size_t(buf.nbytes))
    tr = buf[:C_].astype(np.int64)
    t0 = tr[:, 0].min()
    d = np.diff(tr[:, :7], axis=1)
    for i, nm in enumerate(NAMES):
        print(f"{nm:14s} median {np.median(d[:, i]) / 1e3:7.2f} us  max {d[:, i].max() / 1e3:7.2f} us")
    print(f"block start spread {(tr[:, 0].max() - t0) / 1e3:.2f} us, kernel span {(tr[:, 6].max() - t0) / 1e3:.2f} us")
    if (tr[:, 7] > tr[:, 2]).all() and (tr[:, 2] > tr[:, 1]).all():   # staged fast path stamps
        print(f"fast path: loads {np.median(tr[:, 2] - tr[:, 1]) / 1e3:.2f} us, min/max reduce "
              f"{np.median(tr[:, 7] - tr[:, 2]) / 1e3:.2f} us, keys + arg-min {np.median(tr[:, 3] - tr[:, 7]) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
