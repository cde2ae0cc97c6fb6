"""Host side of the B200 pre-gated MoE block: the reference's types and
operator API (core.py of ``moesim``) over the C ABI of libpgmoe.so.

Two layers:

* ``DeviceModel`` — the product path.  Weights live in HBM (resident) or in
  pinned host memory behind an (L+1)-slot HBM expert cache (offloaded); one
  call runs ``decoder_iteration`` (core.py:342-383) for a whole batch of T
  tokens with K1 (route) / K2 (grouped expert FFN + combine) / K3 (dense)
  on sm_100a and the pre-gated expert migration on a copy stream.
* ``gate_forward`` / ``expert_forward`` / ``moe_block_forward`` /
  ``decoder_iteration`` — drop-ins with the reference signatures
  (core.py:284, :308, :319, :342) that accept the reference's list-based
  ``BlockParams`` / ``ModelParams`` and run the same kernels.

There is no CPU fallback anywhere: without the built library or a CUDA
device every call raises.
"""

from __future__ import annotations

import ctypes
import json
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, RoutingError, ShapeError

# core.py:22-28 substream tags
TAG_GATE, TAG_PRE_GATE, TAG_W1, TAG_W2, TAG_DENSE, TAG_INPUT, TAG_TRACE = range(7)

_DT = {"f32": _lib.F32, "fp32": _lib.F32, "float32": _lib.F32, "bf16": _lib.BF16, "bfloat16": _lib.BF16}
_TORCH_DT = {_lib.F32: torch.float32, _lib.BF16: torch.bfloat16}
_KERNEL = {"auto": _lib.KERNEL_AUTO, "simt": _lib.KERNEL_SIMT, "tcgen05": _lib.KERNEL_TCGEN05}


# --------------------------------------------------------------- types ----

@dataclass(frozen=True)
class ModelConfig:
    """core.py:34-107 — same fields, validation, wiring and sizes."""

    d_model: int
    d_ff: int
    num_blocks: int
    num_experts: int
    top_k: int
    activation_level: int = 1
    dtype_bytes: int = 4
    seed: int = 0
    non_moe_extra_params: int = 0

    def __post_init__(self) -> None:
        for name in ("d_model", "d_ff", "num_blocks", "num_experts", "top_k", "dtype_bytes"):
            v = getattr(self, name)
            if not isinstance(v, int) or v < 1:
                raise ConfigError(f"{name} must be a positive int, got {v!r}")
        if self.top_k > self.num_experts:
            raise ConfigError(f"top_k={self.top_k} exceeds num_experts={self.num_experts}")
        if not 0 <= self.activation_level < self.num_blocks:
            raise ConfigError(f"activation_level={self.activation_level} must be in "
                              f"[0, num_blocks={self.num_blocks})")
        if not 0 <= self.seed <= (1 << 64) - 1:
            raise ConfigError("seed must fit in 64 unsigned bits")
        if self.non_moe_extra_params < 0:
            raise ConfigError("non_moe_extra_params must be >= 0")

    def has_conv_gate(self, block: int) -> bool:
        return True if self.activation_level == 0 else block < self.activation_level

    def has_pre_gate(self, block: int) -> bool:
        return False if self.activation_level == 0 else block < self.num_blocks - self.activation_level

    def decision_origin(self, block: int) -> int:
        if self.activation_level == 0 or block < self.activation_level:
            return block
        return block - self.activation_level

    @property
    def expert_params(self) -> int:
        return 2 * self.d_model * self.d_ff

    @property
    def expert_bytes(self) -> int:
        return self.expert_params * self.dtype_bytes

    @property
    def gate_count(self) -> int:
        return sum(self.has_conv_gate(b) + self.has_pre_gate(b) for b in range(self.num_blocks))

    @property
    def gate_params_each(self) -> int:
        return self.d_model * self.num_experts

    def c_struct(self) -> _lib.Config:
        return _lib.Config(self.d_model, self.d_ff, self.num_blocks, self.num_experts, self.top_k,
                           self.activation_level, self.seed)


@dataclass(frozen=True)
class RoutingDecision:
    """core.py:110-140 — ids by descending logit (ties: lower id)."""

    expert_ids: tuple
    combine_weights: tuple

    def __post_init__(self) -> None:
        if len(self.expert_ids) != len(self.combine_weights):
            raise RoutingError("expert_ids and combine_weights length mismatch")
        if not self.expert_ids:
            raise RoutingError("empty routing decision")
        if len(set(self.expert_ids)) != len(self.expert_ids):
            raise RoutingError(f"duplicate expert ids: {self.expert_ids}")
        for w in self.combine_weights:
            if not (0.0 < w <= 1.0):
                raise RoutingError(f"combine weight {w!r} outside (0, 1]")

    def validate_for(self, config) -> None:
        if len(self.expert_ids) != config.top_k:
            raise RoutingError(f"decision selects {len(self.expert_ids)} experts, "
                               f"model top_k is {config.top_k}")
        for e in self.expert_ids:
            if not 0 <= e < config.num_experts:
                raise RoutingError(f"expert id {e} out of range")


def _stream(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _require_cuda():
    if not torch.cuda.is_available():
        raise _lib.errors.DeviceError("no CUDA device: the B200 path has no CPU fallback")


class DeviceRouting:
    """Device routing buffers for T tokens (pgmoe_routing)."""

    def __init__(self, T: int, E: int, k: int, device="cuda"):
        self.T, self.E, self.k = T, E, k
        n = max(T * k, 1)
        i32 = dict(dtype=torch.int32, device=device)
        self.ids = torch.zeros((T, k), **i32)
        self.w = torch.zeros((T, k), dtype=torch.float32, device=device)
        self.hist = torch.zeros(E, **i32)
        self.off = torch.zeros(E + 1, **i32)
        self.perm = torch.zeros(n, **i32)
        self.w_perm = torch.zeros(n, dtype=torch.float32, device=device)
        self.act_n = torch.zeros(E + 1, **i32)  # act[E] then n_act
        self.status = torch.zeros(4, **i32)
        self.workspace = torch.zeros(_lib.load().pgmoe_route_workspace_bytes(T, E) // 4 + 1, **i32)
        a = self.act_n.data_ptr()
        self._c = _lib.Routing(self.ids.data_ptr(), self.w.data_ptr(), self.hist.data_ptr(),
                               self.off.data_ptr(), self.perm.data_ptr(), self.w_perm.data_ptr(),
                               a, a + 4 * E, self.status.data_ptr(), None)

    @property
    def c(self) -> _lib.Routing:
        return self._c

    @property
    def n_act(self) -> int:
        return int(self.act_n[self.E].item())

    @property
    def act(self) -> torch.Tensor:
        return self.act_n[: self.n_act]

    def check(self) -> dict:
        """Surface device-detected errors (raises) and return counters."""
        fb = ctypes.c_int32(0)
        torch.cuda.synchronize()
        _lib.check(_lib.load().pgmoe_check_routing(ctypes.byref(self._c), ctypes.byref(fb)))
        return {"fallbacks": fb.value}

    def decisions(self) -> list:
        ids = self.ids.cpu().tolist()
        w = self.w.double().cpu().tolist()
        return [RoutingDecision(tuple(i), tuple(x)) for i, x in zip(ids, w)]

    @classmethod
    def from_host(cls, ids: np.ndarray, w: np.ndarray, E: int, device="cuda") -> "DeviceRouting":
        """Build routing buffers from host decisions (supplied/synthetic
        traces, core.py:352-364): the permutation is the same stable
        counting sort K1 produces."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        T, k = ids.shape
        r = cls(T, E, k, device)
        flat = ids.reshape(-1)
        hist = np.bincount(flat, minlength=E).astype(np.int32)
        off = np.zeros(E + 1, dtype=np.int32)
        off[1:] = np.cumsum(hist)
        perm = np.argsort(flat, kind="stable").astype(np.int32)
        act = np.nonzero(hist)[0].astype(np.int32)
        act_n = np.zeros(E + 1, dtype=np.int32)
        act_n[: act.size] = act
        act_n[E] = act.size
        wf = np.ascontiguousarray(w, dtype=np.float32).reshape(-1)
        r.ids.copy_(torch.from_numpy(ids))
        r.w.copy_(torch.from_numpy(wf.reshape(T, k)))
        r.hist.copy_(torch.from_numpy(hist))
        r.off.copy_(torch.from_numpy(off))
        if T:
            r.perm.copy_(torch.from_numpy(perm))
            r.w_perm.copy_(torch.from_numpy(wf[perm]))
        r.act_n.copy_(torch.from_numpy(act_n))
        return r


# ------------------------------------------------------ kernel-level ops --

def route(x: torch.Tensor, gate_w: torch.Tensor, k: int, out: DeviceRouting | None = None,
          stream=None) -> DeviceRouting:
    """K1 on T tokens: x fp32 [T][d] (cuda), gate_w [d][E] fp32/bf16 (cuda);
    or x and gate_w both fp64 — the reference's own precision
    (pgmoe_gate_forward_f64)."""
    _require_cuda()
    if x.dim() == 2 and x.is_cuda and x.dtype == torch.float64 and gate_w.dtype == torch.float64:
        return _route64(x, gate_w, k, out, stream)
    if x.dim() != 2 or x.dtype != torch.float32 or not x.is_cuda:
        raise ShapeError("route expects x as a cuda float32 [T][d] tensor")
    d, E = gate_w.shape
    if k > E:
        raise ConfigError(f"k={k} exceeds expert count {E}")
    if x.shape[1] != d:
        raise ShapeError(f"gate expects input of width {d}, got {x.shape[1]}")
    wdt = _lib.BF16 if gate_w.dtype == torch.bfloat16 else _lib.F32
    T = x.shape[0]
    out = out if out is not None else DeviceRouting(T, E, k, x.device)
    x = x.contiguous()
    gate_w = gate_w.contiguous()
    _lib.check(_lib.load().pgmoe_gate_forward(_ptr(x), T, d, _ptr(gate_w), wdt, E, k, ctypes.byref(out.c),
                                              _ptr(out.workspace), _stream(stream)))
    return out


def _route64(x, gate_w, k, out, stream):
    d, E = gate_w.shape
    if k > E:
        raise ConfigError(f"k={k} exceeds expert count {E}")
    if x.shape[1] != d:
        raise ShapeError(f"gate expects input of width {d}, got {x.shape[1]}")
    T = x.shape[0]
    out = out if out is not None else DeviceRouting(T, E, k, x.device)
    x = x.contiguous()
    gate_w = gate_w.contiguous()
    _lib.check(_lib.load().pgmoe_gate_forward_f64(_ptr(x), T, d, _ptr(gate_w), E, k, ctypes.byref(out.c),
                                                  _ptr(out.workspace), _stream(stream)))
    return out


def expert_ffn(x: torch.Tensor, r: DeviceRouting, experts: torch.Tensor, d_ff: int,
               indexed_by_act: bool = False, kernel: str = "auto", stream=None) -> torch.Tensor:
    """K2: yw [T*k][d] with yw[t*k+s] = w[t,s] * W2 relu(W1 x[t]) of expert ids[t,s].
    experts: [n_records, 2*f*d] (fp32/bf16) — W1 [f][d] then W2 [d][f] per record."""
    T, d = x.shape
    wdt = _lib.BF16 if experts.dtype == torch.bfloat16 else _lib.F32
    stride = experts.stride(0) * experts.element_size()
    h = torch.empty((max(T * r.k, 1), d_ff), dtype=torch.float32, device=x.device)
    yw = torch.empty((max(T * r.k, 1), d), dtype=torch.float32, device=x.device)
    _lib.check(_lib.load().pgmoe_expert_forward(_ptr(x.contiguous()), T, d, d_ff, r.k, _ptr(experts), stride, wdt,
                                                int(indexed_by_act), ctypes.byref(r.c), _ptr(h), _ptr(yw),
                                                _KERNEL[kernel], _stream(stream)))
    return yw[: T * r.k]


def dense(yw: torch.Tensor, T: int, k: int, dense_w: torch.Tensor, kernel: str = "auto",
          stream=None) -> torch.Tensor:
    """K3: y[t] = D . sum_s yw[t*k+s]."""
    d = dense_w.shape[0]
    wdt = _lib.BF16 if dense_w.dtype == torch.bfloat16 else _lib.F32
    y = torch.empty((T, d), dtype=torch.float32, device=yw.device)
    _lib.check(_lib.load().pgmoe_dense_forward(_ptr(yw.contiguous()), T, d, k, _ptr(dense_w.contiguous()), wdt,
                                               _ptr(y), _KERNEL[kernel], _stream(stream)))
    return y


def fill_weights(rows: int, cols: int, seed: int, tag: int, block: int, expert: int = -1,
                 dtype: str = "bf16", device="cuda") -> torch.Tensor:
    """The reference's synthetic matrix (core.py:200-211), generated on the GPU."""
    wdt = _DT[dtype]
    out = torch.empty((rows, cols), dtype=_TORCH_DT[wdt], device=device)
    _lib.check(_lib.load().pgmoe_fill_weights(_ptr(out), wdt, seed, tag, block, expert, rows, cols,
                                              _stream(None)))
    return out


# ------------------------------------------------------------ the model --

class DeviceModel:
    """A pre-gated MoE decoder on one B200 (pgmoe_model)."""

    def __init__(self, config: ModelConfig, dtype: str = "bf16", placement: str = "resident",
                 max_tokens: int = 256, kernel: str = "auto", init: str = "rng", expert_range=None):
        _require_cuda()
        self.config = config
        self.dtype = dtype
        self.wdt = _DT[dtype]
        self.placement = placement
        self.max_tokens = max_tokens
        self._h = ctypes.c_void_p(0)
        self._L = _lib.load()
        c = config.c_struct()
        pl = {"resident": _lib.RESIDENT, "offloaded": _lib.OFFLOADED}[placement]
        e0, e1 = expert_range if expert_range is not None else (0, config.num_experts)
        self.expert_range = (e0, e1)
        _lib.check(self._L.pgmoe_model_create_ex(ctypes.byref(c), self.wdt, pl, max_tokens, e0, e1,
                                                 ctypes.byref(self._h)))
        self.set_kernel(kernel)
        if init == "rng":
            _lib.check(self._L.pgmoe_model_init_weights(self._h))

    def close(self) -> None:
        if self._h:
            self._L.pgmoe_model_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def load(cls, path: str, dtype: str = "bf16", placement: str = "resident", max_tokens: int = 256,
             kernel: str = "auto", seed: int = 0) -> "DeviceModel":
        """model_io.load_model (model_io.py:63-105): a PGMOE1 file into a new model."""
        cfg = weight_file_config(path, seed=seed)
        m = cls(cfg, dtype=dtype, placement=placement, max_tokens=max_tokens, kernel=kernel, init="none")
        _lib.check(m._L.pgmoe_model_load_pgmoe1(m._h, str(path).encode()))
        return m

    def save(self, path: str) -> None:
        """model_io.save_model (model_io.py:39-60): fp32 PGMOE1 file."""
        _lib.check(self._L.pgmoe_model_save_pgmoe1(self._h, str(path).encode()))

    STRATEGIES = {"pre_gated": 0, "on_demand": 1, "prefetch_all": 2}

    def set_strategy(self, strategy: str) -> None:
        """Migration policy of an offloaded model (scheduler.py:36-49)."""
        if strategy not in self.STRATEGIES:
            raise ConfigError(f"unknown strategy {strategy!r}; choose from {sorted(self.STRATEGIES)}")
        _lib.check(self._L.pgmoe_model_set_strategy(self._h, self.STRATEGIES[strategy]))

    CACHE_POLICIES = {"none": 0, "lifo": 1, "lfu": 2, "lru": 3}

    def set_cache(self, policy: str, capacity_fraction: float) -> None:
        """HBM expert cache (cache.py:49-103) of an offloaded model."""
        if policy not in self.CACHE_POLICIES:
            raise ConfigError(f"unknown cache policy {policy!r}; choose from {sorted(self.CACHE_POLICIES)}")
        _lib.check(self._L.pgmoe_model_set_cache(self._h, self.CACHE_POLICIES[policy], float(capacity_fraction)))

    def set_kernel(self, kernel: str) -> None:
        _lib.check(self._L.pgmoe_model_set_kernel(self._h, _KERNEL[kernel]))

    def set_fused_route(self, enabled: bool) -> None:
        """Resident top-1: compute each pre-gate inside the block launch (default)."""
        _lib.check(self._L.pgmoe_model_set_fused_route(self._h, 1 if enabled else 0))

    def set_decode(self, enabled: bool, max_tokens: int = 0) -> None:
        """Resident top-1 at T <= max_tokens (default 1): one persistent launch
        per decoder iteration (pgmoe_model_set_decode)."""
        _lib.check(self._L.pgmoe_model_set_decode(self._h, 1 if enabled else 0, int(max_tokens)))

    def set_ll_decode(self, enabled: bool, max_tokens: int = 0) -> None:
        """Resident, T <= max_tokens (<= 8): the low-latency decoder — one
        persistent launch per decoder iteration whose phases exchange LL
        (flag-in-word) stores (pgmoe_model_set_ll_decode)."""
        _lib.check(self._L.pgmoe_model_set_ll_decode(self._h, 1 if enabled else 0, int(max_tokens)))

    @property
    def ll_decode_iterations(self) -> int:
        return int(self._L.pgmoe_model_ll_decode_iterations(self._h))

    @property
    def decode_iterations(self) -> int:
        return int(self._L.pgmoe_model_decode_iterations(self._h))

    # -- weights (BlockParams `loaded` hook, core.py:185-211) --
    def _mat_shape(self, name):
        c = self.config
        return {"gate": (c.d_model, c.num_experts), "pre_gate": (c.d_model, c.num_experts),
                "w1": (c.d_ff, c.d_model), "w2": (c.d_model, c.d_ff), "non_moe": (c.d_model, c.d_model)}[name]

    def set_matrix(self, name: str, block: int, expert: int, data: np.ndarray) -> None:
        """data in the model dtype: float32, or bf16 bit patterns (uint16)."""
        a = np.ascontiguousarray(data)
        if a.shape != self._mat_shape(name):
            raise ShapeError(f"{name} expects {self._mat_shape(name)}, got {a.shape}")
        _lib.check(self._L.pgmoe_model_set_matrix(self._h, name.encode(), block, expert,
                                                  ctypes.c_void_p(a.ctypes.data), a.nbytes))

    def get_matrix(self, name: str, block: int, expert: int = -1) -> np.ndarray:
        shape = self._mat_shape(name)
        a = np.zeros(shape, dtype=np.uint16 if self.wdt == _lib.BF16 else np.float32)
        _lib.check(self._L.pgmoe_model_get_matrix(self._h, name.encode(), block, expert,
                                                  ctypes.c_void_p(a.ctypes.data), a.nbytes))
        return a

    def matrix(self, name: str, block: int, expert: int = -1) -> torch.Tensor:
        """Zero-copy torch view of a resident matrix (gate/pre_gate/non_moe,
        experts when resident)."""
        p = self._L.pgmoe_model_matrix_ptr(self._h, name.encode(), block, expert)
        if not p:
            raise ConfigError(f"block {block} carries no {name}")
        shape = self._mat_shape(name)
        n = shape[0] * shape[1]
        from torch.utils.dlpack import from_dlpack  # noqa: F401  (documented alternative)
        t = _wrap_device_ptr(p, n, _TORCH_DT[self.wdt])
        return t.view(shape)

    # -- execution --
    def decoder_iteration(self, x: torch.Tensor, trace: bool = False, stream=None, out: torch.Tensor = None,
                          x_trace: torch.Tensor = None, supplied: tuple = None, trace_out: tuple = None):
        """core.py:342-383 for T tokens (x: cuda fp32 [T][d]).
        Returns (y, ids [nb][T][k], w [nb][T][k]) — trace tensors None unless asked.

        x_trace (optional, cuda fp32 [nb][T][d]) receives every block's input.
        supplied = (ids [nb][T][k] int32, w [nb][T][k] fp32) on the device:
        the `supplied_decisions` path (core.py:342-364) — every block
        consumes them and no gate runs.  trace_out = (ids, w) persistent
        trace buffers (instead of fresh ones when trace=True).
        Resident models replay a CUDA graph keyed by the buffer addresses, so
        passing persistent buffers keeps every call on the replay path."""
        c = self.config
        if x.dim() != 2 or x.shape[1] != c.d_model:
            raise ShapeError(f"expected [T][{c.d_model}] input, got {tuple(x.shape)}")
        T = x.shape[0]
        x = x.contiguous()
        y = out if out is not None else torch.empty_like(x)
        ids = w = None
        if trace_out is not None:
            ids, w = trace_out
        elif trace:
            ids = torch.empty((c.num_blocks, T, c.top_k), dtype=torch.int32, device=x.device)
            w = torch.empty((c.num_blocks, T, c.top_k), dtype=torch.float32, device=x.device)
        io = _lib.IterationIO(ids.data_ptr() if ids is not None else None, w.data_ptr() if w is not None else None,
                              None, None, None)
        if x_trace is not None:
            if tuple(x_trace.shape) != (c.num_blocks, T, c.d_model) or x_trace.dtype != torch.float32:
                raise ShapeError(f"x_trace must be float32 [{c.num_blocks}][{T}][{c.d_model}]")
            io.x_trace = x_trace.data_ptr()
        if supplied is not None:
            sid, sw = supplied
            shp = (c.num_blocks, T, c.top_k)
            if tuple(sid.shape) != shp or tuple(sw.shape) != shp or sid.dtype != torch.int32 \
                    or sw.dtype != torch.float32:
                raise ShapeError(f"supplied decisions must be int32 / float32 {shp}")
            io.ids_supplied = sid.contiguous().data_ptr()
            io.w_supplied = sw.contiguous().data_ptr()
        _lib.check(self._L.pgmoe_decoder_iteration_ex(self._h, _ptr(x), T, _ptr(y), ctypes.byref(io),
                                                      _stream(stream)))
        return y, ids, w

    def check_routing(self) -> None:
        """Surface device-detected routing errors of the last iterations
        (GateOverflowError / RoutingError), after a synchronize."""
        _lib.check(self._L.pgmoe_model_check_routing(self._h))

    def decoder_iteration_host(self, x: np.ndarray, trace: bool = False):
        """Same on host buffers (H2D + blocks + D2H inside one C-ABI call)."""
        c = self.config
        x = np.ascontiguousarray(x, dtype=np.float32)
        T = x.shape[0]
        y = np.empty_like(x)
        ids = w = None
        if trace:
            ids = np.empty((c.num_blocks, T, c.top_k), dtype=np.int32)
            w = np.empty((c.num_blocks, T, c.top_k), dtype=np.float32)
        _lib.check(self._L.pgmoe_decoder_iteration_host(
            self._h, ctypes.c_void_p(x.ctypes.data), T, ctypes.c_void_p(y.ctypes.data),
            ctypes.c_void_p(ids.ctypes.data if trace else 0), ctypes.c_void_p(w.ctypes.data if trace else 0)))
        return y, ids, w

    def moe_block_forward(self, block: int, x: torch.Tensor, routing_in: DeviceRouting | None,
                          want_routing_out: bool = True, stream=None):
        """core.py:319-339 for T tokens: (y, routing_out | None)."""
        c = self.config
        T = x.shape[0]
        r_out = None
        if want_routing_out and c.has_pre_gate(block):
            r_out = DeviceRouting(T, c.num_experts, c.top_k, x.device)
        if routing_in is None:
            raise RoutingError("no routing decision available")
        y = torch.empty_like(x)
        _lib.check(self._L.pgmoe_moe_block_forward(
            self._h, block, _ptr(x.contiguous()), T, ctypes.byref(routing_in.c), _ptr(y),
            ctypes.byref(r_out.c) if r_out is not None else None, _stream(stream)))
        return y, r_out

    def stats(self) -> dict:
        s = _lib.Stats()
        _lib.check(self._L.pgmoe_model_stats(self._h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in _lib.Stats._fields_}

    def reset_stats(self) -> None:
        _lib.check(self._L.pgmoe_model_reset_stats(self._h))

    def set_timeline(self, on: bool) -> None:
        _lib.check(self._L.pgmoe_model_set_timeline(self._h, int(on)))

    def timeline(self) -> list:
        n = self._L.pgmoe_model_timeline_jsonl(self._h, None, 0)
        buf = ctypes.create_string_buffer(int(n) + 1)
        self._L.pgmoe_model_timeline_jsonl(self._h, buf, n + 1)
        return [json.loads(line) for line in buf.value.decode().splitlines() if line]


def weight_file_config(path: str, seed: int = 0) -> ModelConfig:
    """Header of a PGMOE1 file (model_io.py:20-21, :70-86) as a ModelConfig."""
    c = _lib.Config()
    _lib.check(_lib.load().pgmoe_weight_file_config(str(path).encode(), ctypes.byref(c)))
    return ModelConfig(d_model=c.d_model, d_ff=c.d_ff, num_blocks=c.num_blocks, num_experts=c.num_experts,
                       top_k=c.top_k, activation_level=c.activation_level, seed=seed)


def _wrap_device_ptr(ptr: int, numel: int, dtype: torch.dtype) -> torch.Tensor:
    """Non-owning torch view of device memory owned by the C library."""
    class _Holder:
        def __init__(self, p, nbytes):
            self.__cuda_array_interface__ = {
                "shape": (nbytes,), "typestr": "|u1", "data": (p, False), "version": 3, "strides": None}
    nbytes = numel * torch.tensor([], dtype=dtype).element_size()
    raw = torch.as_tensor(_Holder(ptr, nbytes), device="cuda")
    return raw.view(dtype)


# ------------------------------------------- drop-ins (reference API) -----

_dev_cache: dict = {}
# The decision type the drop-ins return: this module's RoutingDecision, or —
# once dropin.install() points moesim at these functions — moesim's own.
DECISION_TYPE = RoutingDecision


def clear_cache() -> None:
    _dev_cache.clear()


def _dev_matrix(mat, dtype=torch.float32) -> torch.Tensor:
    """Device copy of a reference list-of-lists matrix (cached by id and
    dtype).  Torch tensors pass through in their own dtype."""
    if isinstance(mat, torch.Tensor):
        return mat.cuda() if not mat.is_cuda else mat
    key = (id(mat), dtype)
    hit = _dev_cache.get(key)
    if hit is not None and hit[0] is mat:
        return hit[1]
    npdt = np.float64 if dtype == torch.float64 else np.float32
    t = torch.tensor(np.asarray(mat, dtype=npdt), device="cuda")
    _dev_cache[key] = (mat, t)
    return t


def _dev_vec(x, dtype=torch.float32) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).reshape(1, -1)
    npdt = np.float64 if dtype == torch.float64 else np.float32
    return torch.tensor(np.asarray(x, dtype=npdt), device="cuda").reshape(1, -1)


def gate_forward(x, gate_weights, k: int) -> RoutingDecision:
    """Drop-in for core.py:284-305 (one token) on the K1 kernel.

    The reference's inputs (Python floats, numpy float64, or fp64 tensors)
    route at fp64 through pgmoe_gate_forward_f64, so ids equal moesim's
    bit-for-bit on its own unrounded init_model weights; fp32 / bf16 tensors
    route through the fp32 kernel (exact products)."""
    if isinstance(gate_weights, torch.Tensor) and gate_weights.dtype != torch.float64:
        G = _dev_matrix(gate_weights)
        xv = _dev_vec(x)
    else:
        G = _dev_matrix(gate_weights, torch.float64)
        xv = _dev_vec(x, torch.float64)
    E = G.shape[1] if G.dim() == 2 and G.shape[0] else 0
    if k > E:
        raise ConfigError(f"k={k} exceeds expert count {E}")
    if G.shape[0] != xv.shape[1]:
        raise ShapeError(f"gate expects input of width {G.shape[0]}, got {xv.shape[1]}")
    r = route(xv, G, k)
    r.check()
    ids = r.ids.cpu().tolist()[0]
    w = r.w.double().cpu().tolist()[0]
    return DECISION_TYPE(tuple(ids), tuple(w))


def expert_forward(x, expert) -> list:
    """Drop-in for core.py:308-316 (one token, one expert) on K2."""
    w1, w2 = _dev_matrix(expert.w1), _dev_matrix(expert.w2)
    xv = _dev_vec(x)
    if w1.shape[1] != xv.shape[1]:
        raise ShapeError(f"expert expects input of width {w1.shape[1]}, got {xv.shape[1]}")
    if w2.shape[1] != w1.shape[0]:
        raise ShapeError("expert w2 width does not match w1 height")
    f, d = w1.shape
    rec = torch.cat([w1.reshape(-1), w2.reshape(-1)]).reshape(1, -1)
    r = DeviceRouting.from_host(np.zeros((1, 1), np.int32), np.ones((1, 1), np.float32), 1)
    yw = expert_ffn(xv, r, rec, f, kernel="simt")
    return yw[0].double().cpu().tolist()


def _block_records(block, ids) -> tuple[torch.Tensor, np.ndarray]:
    uniq = sorted(set(int(e) for e in ids))
    recs = []
    for e in uniq:
        ex = block.expert(e)
        recs.append(torch.cat([_dev_matrix(ex.w1).reshape(-1), _dev_matrix(ex.w2).reshape(-1)]))
    return torch.stack(recs), np.array(uniq, dtype=np.int32)


def moe_block_forward(x, block, routing_in, *, dry_run: bool = False, want_routing_out: bool = True):
    """Drop-in for core.py:319-339 on one token (reference BlockParams)."""
    cfg = block.config
    routing_out = None
    if block.has_pre_gate and (want_routing_out or dry_run):
        routing_out = gate_forward(x, block.pre_gate, cfg.top_k)
    if dry_run:
        return None, routing_out
    if routing_in is None:
        raise RoutingError("no routing decision available")
    routing_in.validate_for(cfg)
    xv = _dev_vec(x)
    recs, uniq = _block_records(block, routing_in.expert_ids)
    # slot-indexed records: position of each expert in the ascending active list
    r = DeviceRouting.from_host(np.array([routing_in.expert_ids], np.int32),
                                np.array([routing_in.combine_weights], np.float32), cfg.num_experts)
    yw = expert_ffn(xv, r, recs, cfg.d_ff, indexed_by_act=True, kernel="simt")
    y = dense(yw, 1, cfg.top_k, _dev_matrix(block.non_moe), kernel="simt")
    return y[0].double().cpu().tolist(), routing_out


def decoder_iteration(x, params, supplied_decisions=None):
    """Drop-in for core.py:342-383 (one token, reference ModelParams)."""
    cfg = params.config
    if supplied_decisions is not None:
        if len(supplied_decisions) != cfg.num_blocks:
            raise RoutingError(f"supplied {len(supplied_decisions)} decisions for {cfg.num_blocks} blocks")
        for d in supplied_decisions:
            d.validate_for(cfg)
    pending: dict = {}
    consumed = []
    for b in range(cfg.num_blocks):
        block = params.blocks[b]
        if supplied_decisions is not None:
            decision = supplied_decisions[b]
        elif cfg.has_conv_gate(b):
            decision = gate_forward(x, block.gate, cfg.top_k)
        else:
            try:
                decision = pending.pop(b)
            except KeyError:
                raise RoutingError(f"no routing decision available for block {b}") from None
        x, routing_out = moe_block_forward(x, block, decision, want_routing_out=supplied_decisions is None)
        if routing_out is not None:
            target = b + cfg.activation_level
            if target in pending:
                raise RoutingError(f"duplicate decision emitted for block {target}")
            pending[target] = routing_out
        consumed.append(decision)
    if pending:
        raise RoutingError(f"unconsumed decisions for blocks {sorted(pending)}")
    return x, consumed


def token_inputs(config: ModelConfig, T: int, offset: int = 0, device="cuda") -> torch.Tensor:
    """Synthetic batch: token 0 = default_input (core.py:274),
    token t>=1 = Xoshiro(derive_seed(seed, 5, t)).fill(d); rounded to fp32."""
    from ._rng import token_batch
    return torch.from_numpy(token_batch(config.seed, config.d_model, T, offset)).to(device)
