"""B200-native pre-gated MoE block (arXiv 2308.12066) behind the reference
``moesim`` block API.  See DESIGN.md / INTEGRATION.md."""

from .errors import (ConfigError, DeviceError, GateOverflowError, InvariantError, MoESimError,
                     OomError, RoutingError, ShapeError, WeightFileError)

__version__ = "0.1.0"

_CORE_NAMES = ("ModelConfig", "RoutingDecision", "DeviceModel", "DeviceRouting", "route", "expert_ffn",
               "dense", "fill_weights", "gate_forward", "expert_forward", "moe_block_forward",
               "decoder_iteration", "token_inputs", "clear_cache", "weight_file_config")


def __getattr__(name):  # torch is imported lazily so the package imports without it
    if name in _CORE_NAMES:
        from . import core
        return getattr(core, name)
    raise AttributeError(name)


__all__ = ["ConfigError", "DeviceError", "GateOverflowError", "InvariantError", "MoESimError", "OomError",
           "RoutingError", "ShapeError", "WeightFileError", *_CORE_NAMES]
