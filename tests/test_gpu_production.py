"""GPU parity of the PRODUCTION step path (the one bench.py times): attention without the
weights dump (WD=false combines), K1 forked beside it, K3/K4 writing the kept-index map,
replayed from one captured CUDA graph. Each step the weights-dumping attention runs first and
feeds the oracle; the production step must reproduce its staged head mean and its output bit
for bit, so every oracle check (kept sets, EMA, codes, records; attention at 1e-3) covers the
production kernels. K2's launch-size rules are also forced both ways on small scenarios
(CKV_COMB: k2_combine<1> / k2_combine<4> / k2_combine_staged; CKV_DYN: static-stride or
dynamically claimed items in the persistent tcgen05 grid; CKV_TC: that grid on / off;
CKV_FSTREAM: the FP16 parts on the persistent streaming kernel or on the general kernel)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import scenarios as S  # noqa: E402
from tests.gpu_driver import run_scenario  # noqa: E402

SMALL = [n for n in S.SCENARIOS if n not in ("gpt2_c1", "niah_32k")]


@pytest.mark.parametrize("name", SMALL)
def test_production_graph_path(name):
    r = run_scenario(name, batch=2, steps=min(S.SCENARIOS[name]["steps"], 40), check_every=20,
                     production=True, graph=True)
    assert r["worst_attn_rel"] < 1e-3


@pytest.mark.parametrize("comb", ["plain1", "plain4", "staged"])
@pytest.mark.parametrize("dyn", ["static", "dynamic"])
@pytest.mark.parametrize("name", ["int8_bulk_d128", "gqa5_int8_d128", "int8_d128_long", "absorb_int8_d128"])
def test_forced_k2_paths_int8(name, comb, dyn, monkeypatch):
    monkeypatch.setenv("CKV_COMB", comb)
    monkeypatch.setenv("CKV_DYN", dyn)
    monkeypatch.setenv("CKV_TC", "on")
    r = run_scenario(name, batch=2, steps=10, check_every=5, production=True, graph=True)
    assert r["worst_attn_rel"] < 1e-3


@pytest.mark.parametrize("fstream", ["0", "1"])
@pytest.mark.parametrize("tc", ["on", "off"])
@pytest.mark.parametrize("name", ["int8_bulk_d128", "gqa5_int8_d128", "int8_d128_long", "absorb_int8_d128",
                                  "fp16_d128_long", "absorb_fp16_d128", "gqa8_int8_d64", "fp16_mha", "int8_mha",
                                  "pyramid_gqa"])
def test_forced_fp16_stream(name, tc, fstream, monkeypatch):
    """The FP16 streaming kernel (k2_fp16_stream: one warp per (cache, KV head, FP16 part),
    per-warp rings fed across units) forced on / off beside the tcgen05 grid on / off, so its
    partial slots, scores and the cut-mode codes parts of the general kernel meet the oracle on
    small scenarios (the default launch rules use it only for big launches)."""
    monkeypatch.setenv("CKV_FSTREAM", fstream)
    monkeypatch.setenv("CKV_TC", tc)
    r = run_scenario(name, batch=2, steps=10, check_every=5, production=True, graph=True)
    assert r["worst_attn_rel"] < 1e-3


@pytest.mark.parametrize("comb", ["plain1", "plain4", "staged"])
@pytest.mark.parametrize("name", ["fp16_d128_long", "absorb_fp16_d128", "gqa8_int8_d64", "fp16_mha", "int8_mha"])
def test_forced_combines(name, comb, monkeypatch):
    monkeypatch.setenv("CKV_COMB", comb)
    r = run_scenario(name, batch=2, steps=12, check_every=6, production=True, graph=True)
    assert r["worst_attn_rel"] < 1e-3


@pytest.mark.parametrize("name", ["int8_mha", "pyramid_gqa", "int8_bulk_d128", "gqa8_int8_d64", "fp16_mha",
                                  "edge_alpha0_temp", "edge_p0_w0"])
def test_forced_k3_256(name, monkeypatch):
    """K3 as 256-thread CTAs (launch_manage picks them for many short caches, e.g. the Qwen-32B
    pyramid's 512): kept maps, EMA, codes and records against the oracle."""
    monkeypatch.setenv("CKV_K3T", "256")
    r = run_scenario(name, batch=2, steps=12, check_every=6, production=True, graph=True)
    assert r["worst_attn_rel"] < 1e-3


def test_niah_production_path():
    """C4 step 1 (32,768 entries, 32K -> 512 select, bulk demotion) eager, then the graph."""
    r = run_scenario("niah_32k", batch=1, steps=6, check_every=6, production=True, graph=True)
    assert r["worst_attn_rel"] < 1e-3


def test_gpt2_c1_all_512_steps():
    """C1 at its real shape (GPT-2 small: L=12, H=12, D=64, V=50,257), batch 1, 512-entry
    prefill, all 512 decode steps on the production graph path: kept sets, EMA bits, records
    bit-exact against the oracle (pinned to the reference by engine_gpt2_c1 fixtures), attention
    at 1e-3. Also counts the decisions where the reference's own fp64 attention would keep a
    different set than the GPU's fp32 attention (0/512 on the CPU)."""
    r = run_scenario("gpt2_c1", batch=1, check_every=128, production=True, graph=True,
                     own_attention_trials=True)
    assert r["steps"] == 512 and r["worst_attn_rel"] < 1e-3
    print(f"C1 kept-set mismatches vs the reference's own fp64 attention: "
          f"{r['kept_mismatch']} / {r['kept_trials']} (step, layer) decisions")
    assert r["kept_trials"] == 512 * 12
    assert r["kept_mismatch"] <= r["kept_trials"] // 100
