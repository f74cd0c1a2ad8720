"""Phase timing of K2's tcgen05 INT8 path from a -DCKV_TRACE build (debug tool, GPU box).

  CKV_NVCC_EXTRA=-DCKV_TRACE python -m paper_2605_24786_b200.build --force
  python tools/trace_k2.py [--workload llama8b_int8_4k]

Sets up the bench workload, runs a few steps, then one more attend_layers() whose CTAs stamp
%globaltimer at each phase boundary; prints per-phase medians and per-SM CTA concurrency.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

NAMES = ["entry", "rows+decide", "bar init", "K issue+Qd", "QK0", "QK1", "QK2", "QK3", "max sync",
         "P+PV issue", "last PV", "O epilogue"]


def main():
    import torch
    import bench
    from paper_2605_24786_b200 import _lib
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
        v = torch.randn((1, B, n, Hkv, D), generator=g, device=dev).half()
        eng.prefill(k, v, layer_begin=layer)
    q = torch.randn((L, B, H, D), generator=g, device=dev).half()
    for t in range(1, 6):
        logits = torch.randn((B, V), generator=g, device=dev) * 8
        kn = torch.randn((L, B, Hkv, D), generator=g, device=dev).half()
        eng.attend_layers(q)
        eng.step(logits, kn, kn, step=t, kept=False)
    torch.cuda.synchronize()
    eng.attend_layers(q)
    torch.cuda.synchronize()
    lib = _lib.load()
    buf = np.zeros((32768, 16), dtype=np.uint64)
    lib.ckv_debug_trace.restype = C.c_int
    rc = lib.ckv_debug_trace(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
    assert rc == 0, rc
    t0 = buf[:, 0].astype(np.int64)
    live = t0 > 0
    base = t0[live].min()
    tc = live & (buf[:, 11] > buf[:, 0]) & (buf[:, 2] > buf[:, 0])
    print(f"CTAs stamped {live.sum()}, tcgen05 path {tc.sum()}")
    x = buf[tc].astype(np.int64)
    span = (buf[live, 0].astype(np.int64).max() - base) / 1e3
    print(f"launch span (first entry .. last entry) {span:.1f} us; last tc end {(x[:, 11].max() - base) / 1e3:.1f} us")
    prev = x[:, 0]
    for i in range(1, 12):
        cur = x[:, i]
        d = (cur - prev) / 1e3
        print(f"  {NAMES[i]:>12}: median {np.median(d):7.2f} us  p90 {np.percentile(d, 90):7.2f}  mean {d.mean():7.2f}")
        prev = cur
    tot = (x[:, 11] - x[:, 0]) / 1e3
    print(f"  {'total':>12}: median {np.median(tot):7.2f} us  p90 {np.percentile(tot, 90):7.2f}")
    # concurrency: average number of tc CTAs resident per SM over the launch
    sm = buf[tc, 15].astype(np.int64)
    busy = np.zeros(256)
    for s in np.unique(sm):
        busy[s] = tot[sm == s].sum()
    active = busy[busy > 0]
    print(f"  SMs with tc CTAs {len(active)}; tc CTA-us per SM median {np.median(active):.0f} "
          f"-> mean tc CTAs resident {np.median(active) / span:.2f}")
    gen = live & ~tc
    print(f"  general-path CTAs {gen.sum()} (decide at median {np.median((buf[gen,1]-buf[gen,0]).astype(np.int64))/1e3:.2f} us)")


if __name__ == "__main__":
    main()
