"""B200-native Conf-KV per-decode-step cache manager (arxiv 2605.24786).

Host side: `config` (drop-in PolicyConfig / ModelShape / presets) and
`engine.ConfKVEngine` (drop-in for confkv.policy.ConfKVEngine, batched).
Device side: hand-written sm_100a kernels behind the C ABI in
include/confkv_b200.h, built by `python -m paper_2605_24786_b200.build`.
"""

from .config import (PRESETS, ConfigError, ModelShape, PolicyConfig, budget_table, load_config,
                     preset, pyramid_budget)

__version__ = "0.1.0"


def __getattr__(name):
    # the engine needs torch + CUDA + the built library; import lazily so the
    # host-only config API stays importable everywhere
    if name in ("ConfKVEngine", "StepRecord", "StepResult"):
        from . import engine
        return getattr(engine, name)
    raise AttributeError(name)


__all__ = ["ConfigError", "ModelShape", "PolicyConfig", "PRESETS", "preset", "load_config",
           "pyramid_budget", "budget_table", "ConfKVEngine", "StepRecord", "StepResult"]
