import os, sys
sys.path.insert(0, os.getcwd())
from oracle import scenarios as S
from tests.gpu_driver import run_scenario
S.SCENARIOS["tmp_short"] = dict(L=2, H=8, Hkv=2, D=128, V=700, prefill=40, steps=40, quantize=True,
    cfg=dict(n_high=96, n_low=160, protected_p=16, pyramid_n_min=96, fp16_window_w=32, alpha=0.7), seed=5)
try:
    print(run_scenario("tmp_short", batch=3, check_every=5))
except AssertionError as e:
    print("FAIL", str(e)[:500])
