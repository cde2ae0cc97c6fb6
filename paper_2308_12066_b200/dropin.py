"""Install the B200 path into an unmodified ``moesim`` (the reference package).

``install()`` points moesim's hot-path names — ``gate_forward``
(core.py:284-305), ``expert_forward`` (core.py:308-316), ``moe_block_forward``
(core.py:319-339) and ``decoder_iteration`` (core.py:342-383) — at this
package's drop-ins, which run K1 / K2 / K3 on the sm_100a kernels through the
C ABI.  ``scheduler.py:29-30`` and ``harness.py:18`` bind
``decoder_iteration`` by name at import, so those modules are patched too.

Inside moesim the drop-ins speak moesim's own types: decisions are
``moesim.core.RoutingDecision`` instances and errors are raised as the
same-named ``moesim.errors`` classes with the reference messages, so
moesim's callers (``simulate``, the harness's ``verify_result``) and its
tests see no difference but the device.

    from paper_2308_12066_b200 import dropin
    handle = dropin.install()          # import moesim, patch it
    ...                                # moesim.simulate(...) runs its math pass on the GPU
    handle.uninstall()

There is no CPU fallback: without the built library or a CUDA device the
first call raises.
"""

from __future__ import annotations

import functools
import importlib

from . import core as _core
from . import errors as _errors

HOT_PATH = ("gate_forward", "expert_forward", "moe_block_forward", "decoder_iteration")
# modules that hold their own reference to a hot-path name (bound at import)
PATCHED_MODULES = ("moesim.core", "moesim.scheduler", "moesim.harness", "moesim")


def _translate(fn, ref_errors):
    """Re-raise this package's exceptions as moesim's same-named classes."""
    ours = {getattr(_errors, n): getattr(ref_errors, n) for n in
            ("ConfigError", "ShapeError", "GateOverflowError", "RoutingError", "OomError", "WeightFileError",
             "InvariantError", "MoESimError") if hasattr(ref_errors, n)}

    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except _errors.MoESimError as e:
            for cls in type(e).__mro__:
                if cls in ours:
                    raise ours[cls](str(e)) from e
            raise
    return wrapper


class Installation:
    """What install() changed, so that uninstall() can restore it."""

    def __init__(self):
        self.saved: list = []  # (module, name, original)
        self.decision_type = _core.DECISION_TYPE

    def uninstall(self) -> None:
        for mod, name, orig in reversed(self.saved):
            setattr(mod, name, orig)
        self.saved.clear()
        _core.DECISION_TYPE = self.decision_type
        _core.clear_cache()


def install(package: str = "moesim") -> Installation:
    """Patch an importable moesim so its hot path runs on the B200 kernels."""
    ref_core = importlib.import_module(f"{package}.core")
    ref_errors = importlib.import_module(f"{package}.errors")
    inst = Installation()
    _core.DECISION_TYPE = ref_core.RoutingDecision
    for modname in PATCHED_MODULES:
        modname = modname.replace("moesim", package, 1)
        try:
            mod = importlib.import_module(modname)
        except ImportError:
            continue
        for name in HOT_PATH:
            if hasattr(mod, name):
                inst.saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, _translate(getattr(_core, name), ref_errors))
    return inst
