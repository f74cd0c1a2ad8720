"""Per-item phase timing of K2's persistent tcgen05 kernel from a -DCKV_TRACE build (debug
tool, GPU box).

  CKV_NVCC_EXTRA=-DCKV_TRACE python -m paper_2605_24786_b200.build --force
  python tools/trace_k2p.py [--workload llama8b_int8_4k]

Runs the bench workload's steady state, then one more all-layer attend whose persistent CTAs
stamp clock64 at 12 role events per item (first 64 items per CTA); prints median intervals.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

EV = ["P rows start", "P item published", "P last chunk issued", "M item seen", "M Qd+TMEM ready",
      "M QK issued", "M PV issued (O commit)", "E item seen", "E Qd done", "E scores+max done",
      "E O ready", "E item end"]


def main():
    import torch
    import bench
    from paper_2605_24786_b200 import _lib
    from paper_2605_24786_b200.config import ModelShape, PolicyConfig
    from paper_2605_24786_b200.engine import ConfKVEngine

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama8b_int8_4k")
    ap.add_argument("--mhz", type=float, default=1965.0)
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
    lib = _lib.load()
    buf = np.zeros((512, 64, 12), dtype=np.int64)
    lib.ckv_debug_ptrace.restype = C.c_int
    lib.ckv_debug_ptrace(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))  # clear below
    buf[:] = 0
    zero = np.zeros_like(buf)
    # zero the device buffer by copying zeros in through a fresh launch is not possible from
    # the ABI; instead compare before/after: stamps of this launch are the ones that changed
    before = np.zeros_like(buf)
    lib.ckv_debug_ptrace(before.ctypes.data_as(C.c_void_p), C.c_size_t(before.nbytes))
    eng.attend_layers(q)
    torch.cuda.synchronize()
    lib.ckv_debug_ptrace(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
    fresh = (buf != before).all(axis=2)          # items fully re-stamped by this launch
    us = 1.0 / a.mhz
    print(f"CTAs with items {int(fresh.any(axis=1).sum())}, items traced {int(fresh.sum())}")

    def med(name, x):
        x = np.asarray(x, dtype=np.float64) * us
        if x.size:
            print(f"  {name:>34}: median {np.median(x):7.2f} us  p10 {np.percentile(x, 10):7.2f}  p90 {np.percentile(x, 90):7.2f}")

    iv = {k: [] for k in ["Prows", "Pissue", "Pwait", "Mwait_qd", "MQK", "MPV", "Midle", "EQd", "Escores",
                          "EP_waitO", "EOepi", "Eperiod", "Egap", "pub_vs_end"]}
    for cta in range(512):
        js = np.nonzero(fresh[cta])[0]
        for j in js:
            r = buf[cta, j]
            iv["Prows"].append(r[1] - r[0]); iv["Pissue"].append(r[2] - r[1])
            iv["Mwait_qd"].append(r[4] - r[3]); iv["MQK"].append(r[5] - r[4]); iv["MPV"].append(r[6] - r[5])
            iv["EQd"].append(r[8] - r[7]); iv["Escores"].append(r[9] - r[8])
            iv["EP_waitO"].append(r[10] - r[9]); iv["EOepi"].append(r[11] - r[10])
            if j + 1 < 64 and fresh[cta, j + 1]:
                r2 = buf[cta, j + 1]
                iv["Pwait"].append(r2[0] - r[2]); iv["Midle"].append(r2[3] - r[6])
                iv["Eperiod"].append(r2[11] - r[11]); iv["Egap"].append(r2[7] - r[11])
                iv["pub_vs_end"].append(r2[1] - r[11])
    names = {"Prows": "producer: rows lookup", "Pissue": "producer: chunk issue (incl. slot waits)",
             "Pwait": "producer: wait item buffer", "Mwait_qd": "MMA: wait Qd / TMEM",
             "MQK": "MMA: QK issue (incl. K waits)", "MPV": "MMA: PV issue (incl. P/V waits)",
             "Midle": "MMA: idle to next item", "EQd": "epi: Qd digits", "Escores": "epi: scores + max",
             "EP_waitO": "epi: P digits + wait O", "EOepi": "epi: O epilogue", "Eperiod": "item period",
             "Egap": "epi: end -> next item seen", "pub_vs_end": "next item published - epi end"}
    for k, v in iv.items():
        med(names[k], v)


if __name__ == "__main__":
    main()
