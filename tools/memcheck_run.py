"""compute-sanitizer driver (GPU box): production-path steps of small scenarios through the
kernels r02 added or changed -- the FP16 streaming kernel with FP16 and codes units, beside and
without the tcgen05 grid (the latter behind the one-wave general grid), the K3 staged fast path
with its single-victim free and K/V append at 512 and 256 threads, K4's early exit, K1 -- checked
against the oracle as usual.

  compute-sanitizer --tool memcheck python tools/memcheck_run.py   (profiles/r02_memcheck.txt)
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from tests.gpu_driver import run_scenario  # noqa: E402

CFGS = [("int8_bulk_d128", {"CKV_TC": "off", "CKV_FSTREAM": "1"}),
        ("gqa5_int8_d128", {"CKV_TC": "on", "CKV_FSTREAM": "1"}),
        ("fp16_d128_long", {"CKV_FSTREAM": "1"}),
        ("pyramid_gqa", {}),
        ("int8_mha", {}),
        ("int8_mha", {"CKV_K3T": "256"}),
        ("edge_p0_w0", {"CKV_K3T": "256"})]

if __name__ == "__main__":
    for name, env in CFGS:
        os.environ.update(env)
        r = run_scenario(name, batch=2, steps=6, check_every=3, production=True, graph=False)
        print(name, env, r["worst_attn_rel"])
        for k in env:
            os.environ.pop(k)
