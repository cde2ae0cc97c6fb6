"""Expert parallelism (BASELINE configs[4]).

Experts of every block are partitioned contiguously over P ranks (one
process per GPU, ``torch.distributed``); gates and dense layers are
replicated; every rank owns its own T sequences.  Per block there is
exactly one exchange step each way:

  K1 route (local tokens) -> counts [P][E/P] all-to-all -> dispatch rows
  (all_to_all_single, NCCL over NVLink) -> receiver routing + K2 on the
  local experts -> combine rows back -> weighted un-permute -> K3 dense.

Because K1's permutation is grouped by expert and experts are contiguous
per rank, the packed send buffer is already grouped by destination; the
receiver regroups its rows by local expert with the same stable order a
single GPU would use, so EP outputs equal the single-GPU outputs.

With bf16 weights on the tcgen05 path the exchange is FIXED-SIZE: every
rank reserves a slot of cap = T*k rows for every peer, so both all-to-alls
run with equal splits and the host never waits for split sizes (no device
-> host round trip per block); rows travel as the bf16 operand the FFN
consumes (exact, half the bytes), results come back in fp32 for the exact
combine.  The split-size variant (``Exchange.rows``) remains for the fp32
SIMT path.

The exchange plans (``dispatch_plan``/``local_routing_plan`` and their
padded forms) and the collectives (``Exchange``) are backend-neutral and are
exercised on CPU with gloo in tests/test_ep_gloo.py; ``EPDecoder`` drives
them with the sm_100a kernels.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .core import DeviceRouting, ModelConfig, _ptr, _stream
from .errors import DeviceError, ConfigError, ShapeError


def expert_range(E: int, P: int, rank: int) -> tuple[int, int]:
    if E % P:
        raise ConfigError(f"num_experts={E} is not divisible by world size {P}")
    el = E // P
    return rank * el, (rank + 1) * el


def dispatch_plan(hist: np.ndarray, P: int) -> tuple[np.ndarray, np.ndarray]:
    """hist [E] (tokens per global expert, this rank) -> (per-expert counts
    [P][E/P] sent to each rank, rows sent to each rank [P])."""
    h = np.asarray(hist).reshape(P, -1)
    return h, h.sum(axis=1)


def local_routing_plan(recv_cnt: np.ndarray):
    """Host restatement of pgmoe_ep_local_routing: recv_cnt [P][El] ->
    (hist [El], off [El+1], perm [n]) over the received rows."""
    P, El = recv_cnt.shape
    src_base = np.concatenate([[0], np.cumsum(recv_cnt.sum(axis=1))[:-1]])
    src_off = np.concatenate([np.zeros((P, 1), np.int64), np.cumsum(recv_cnt, axis=1)[:, :-1]], axis=1)
    hist = recv_cnt.sum(axis=0)
    off = np.concatenate([[0], np.cumsum(hist)])
    perm = []
    for e in range(El):
        for p in range(P):
            b = src_base[p] + src_off[p, e]
            perm.extend(range(b, b + recv_cnt[p, e]))
    return hist.astype(np.int32), off.astype(np.int32), np.array(perm, dtype=np.int32)


def padded_send_plan(hist: np.ndarray, P: int, cap: int) -> np.ndarray:
    """Slot of every routing position r in the fixed-size send buffer
    (rank p's slot starts at p*cap): host restatement of pgmoe_ep_pack_send."""
    h = np.asarray(hist)
    El = h.size // P
    off = np.concatenate([[0], np.cumsum(h)])
    slot = np.empty(int(off[-1]), dtype=np.int64)
    for p in range(P):
        a, b = off[p * El], off[(p + 1) * El]
        slot[a:b] = p * cap + np.arange(b - a)
    return slot


def local_routing_plan_padded(recv_cnt: np.ndarray, cap: int):
    """pgmoe_ep_local_routing_padded: like local_routing_plan, source p's rows
    start at p*cap."""
    P, El = recv_cnt.shape
    src_off = np.concatenate([np.zeros((P, 1), np.int64), np.cumsum(recv_cnt, axis=1)[:, :-1]], axis=1)
    hist = recv_cnt.sum(axis=0)
    off = np.concatenate([[0], np.cumsum(hist)])
    perm = []
    for e in range(El):
        for p in range(P):
            b = p * cap + src_off[p, e]
            perm.extend(range(b, b + recv_cnt[p, e]))
    return hist.astype(np.int32), off.astype(np.int32), np.array(perm, dtype=np.int32)


class Exchange:
    """The two all-to-all steps of a block, over a torch.distributed group
    (NCCL for device tensors; gloo works for CPU tensors)."""

    def __init__(self, group=None):
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def counts(self, send_cnt: torch.Tensor) -> torch.Tensor:
        """send_cnt [P][El] int32 -> recv_cnt [P][El] (row p = from rank p)."""
        recv = torch.empty_like(send_cnt)
        dist.all_to_all_single(recv, send_cnt.contiguous(), group=self.group)
        return recv

    def fixed(self, send: torch.Tensor, recv: torch.Tensor) -> torch.Tensor:
        """Equal-split all-to-all (rank p's chunk = rows [p*cap, (p+1)*cap))."""
        dist.all_to_all_single(recv, send, group=self.group)
        return recv

    def rows(self, send: torch.Tensor, send_splits: list, recv_splits: list) -> torch.Tensor:
        out = send.new_empty((int(sum(recv_splits)),) + tuple(send.shape[1:]))
        dist.all_to_all_single(out, send, output_split_sizes=[int(v) for v in recv_splits],
                               input_split_sizes=[int(v) for v in send_splits], group=self.group)
        return out


class EPDecoder:
    """decoder_iteration (core.py:342-383) with experts sharded over ranks."""

    def __init__(self, config: ModelConfig, dtype: str = "bf16", max_tokens: int = 256, group=None,
                 kernel: str = "auto"):
        from .core import DeviceModel
        self.config = config
        self.ex = Exchange(group)
        self.P, self.rank = self.ex.P, self.ex.rank
        self.e0, self.e1 = expert_range(config.num_experts, self.P, self.rank)
        self.El = self.e1 - self.e0
        self.model = DeviceModel(config, dtype=dtype, placement="resident", max_tokens=max_tokens,
                                 kernel=kernel, init="rng", expert_range=(self.e0, self.e1))
        self.kernel = kernel
        self.max_tokens = max_tokens
        k = config.top_k
        self.max_recv = self.P * max_tokens * k
        self.lr = DeviceRouting(self.max_recv, self.El, 1)
        self.routing = DeviceRouting(max_tokens, config.num_experts, k)
        self._L = _lib.load()
        self.timing = {"exchange_s": 0.0, "blocks": 0}
        # benchmark hook: (start, end, n_act tensor) CUDA events around each
        # expert FFN launch of an eager iteration (None: off)
        self.ffn_events = None
        import os
        self.use_graph = os.environ.get("PGMOE_EP_GRAPH", "1") != "0"
        self._graphs: dict = {}
        self.replayed_kernels = 0  # our kernels launched by graph replays (benchmark evidence)
        self._side = torch.cuda.Stream()  # the pre-gates (off the critical path)
        self._rbufs: dict = {}
        # fixed-size exchange buffers (tcgen05 path): slot of cap rows per peer
        self.packed = dtype == "bf16" and kernel != "simt" and config.d_model % 128 == 0 \
            and config.d_ff % 128 == 0 and config.d_ff >= config.d_model
        self.cap = max_tokens * k
        if self.packed:
            dev = torch.device("cuda", torch.cuda.current_device())
            rows, d, f = self.P * self.cap, config.d_model, config.d_ff
            # per-peer slot: cap rows + a header carrying the counts (one
            # all-to-all moves both)
            self.slot = int(self._L.pgmoe_ep_slot_rows(self.cap, self.El, d))
            srows = self.P * self.slot
            bf = dict(dtype=torch.bfloat16, device=dev)
            self.send = torch.zeros((srows, d), **bf)
            self.recv = torch.zeros((srows, d), **bf)
            self.xb = torch.zeros((rows, d), **bf)
            self.hb = torch.zeros((rows, f), **bf)
            self.y_recv = torch.zeros((srows, d), dtype=torch.float32, device=dev)
            self.back = torch.zeros((srows, d), dtype=torch.float32, device=dev)
            self.yw = torch.zeros((self.cap, d), dtype=torch.float32, device=dev)
            self.mixb = torch.zeros((max_tokens, d), **bf)

    def block(self, b: int, x: torch.Tensor, r_in: DeviceRouting, stream=None):
        if self.packed:
            return self._block_fixed(b, x, r_in, stream)
        return self._block_splits(b, x, r_in, stream)

    def _block_fixed(self, b: int, x: torch.Tensor, r_in: DeviceRouting, stream=None):
        """One block with the fixed-size exchange: no host synchronisation."""
        c, L, ex = self.config, self._L, self.ex
        T, d, f, k = x.shape[0], c.d_model, c.d_ff, c.top_k
        P, El, cap = self.P, self.El, self.cap
        if T * k > cap:
            raise ShapeError(f"T={T} exceeds the EP buffers (max_tokens={self.max_tokens})")
        s = _stream(stream)
        _lib.check(L.pgmoe_ep_pack_send(_ptr(x), ctypes.byref(r_in.c), T, d, k, P, El, cap, _ptr(self.send), s))
        ex.fixed(self.send, self.recv)                   # bf16 rows + counts header, one slot per peer
        # receiver routing + rows packed in local-expert order, one launch
        _lib.check(L.pgmoe_ep_recv_route_pack(_ptr(self.recv), P, El, cap, d, ctypes.byref(self.lr.c),
                                              _ptr(self.xb), s))
        base, stride = ctypes.c_void_p(), ctypes.c_size_t()
        eb, nl = ctypes.c_int32(), ctypes.c_int32()
        _lib.check(L.pgmoe_model_expert_records(self.model._h, b, ctypes.byref(base), ctypes.byref(stride),
                                                ctypes.byref(eb), ctypes.byref(nl)))
        ev = None
        if self.ffn_events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record(torch.cuda.current_stream() if stream is None else stream)
        _lib.check(L.pgmoe_expert_forward_packed(_ptr(self.xb), P * cap, d, f, base, stride.value,
                                                 ctypes.byref(self.lr.c), _ptr(self.hb), _ptr(self.y_recv), s))
        if ev is not None:
            ev[1].record(torch.cuda.current_stream() if stream is None else stream)
            self.ffn_events.append((ev[0], ev[1], self.lr.act_n[El:El + 1].clone()))
        ex.fixed(self.y_recv, self.back)                 # fp32 results back to their senders
        y = torch.empty_like(x)
        if k == 1:  # combine straight into the dense layer's bf16 operand (as the fused single-GPU epilogue)
            _lib.check(L.pgmoe_ep_unpermute_padded_bf16(_ptr(self.back), ctypes.byref(r_in.c), T, d, P, El, cap,
                                                        _ptr(self.mixb), s))
            _lib.check(L.pgmoe_dense_forward_packed(_ptr(self.mixb), T, d, _ptr(self.model.matrix("non_moe", b)),
                                                    _ptr(y), s))
            return y
        _lib.check(L.pgmoe_ep_unpermute_padded(_ptr(self.back), ctypes.byref(r_in.c), T, d, k, P, El, cap,
                                               _ptr(self.yw), s))
        from .core import _KERNEL
        _lib.check(L.pgmoe_dense_forward(_ptr(self.yw), T, d, k, _ptr(self.model.matrix("non_moe", b)),
                                         self.model.wdt, _ptr(y), _KERNEL[self.kernel], s))
        return y

    def _block_splits(self, b: int, x: torch.Tensor, r_in: DeviceRouting, stream=None):
        c = self.config
        L = self._L
        T, d, f, k = x.shape[0], c.d_model, c.d_ff, c.top_k
        n = T * k
        hist2 = r_in.hist.view(self.P, self.El)
        recv_cnt = self.ex.counts(hist2)                      # [P][El] exchange (one block early in principle)
        splits = torch.stack([hist2.sum(1), recv_cnt.sum(1)]).cpu()
        send_splits, recv_splits = splits[0].tolist(), splits[1].tolist()
        x_send = torch.empty((max(n, 1), d), dtype=torch.float32, device=x.device)
        _lib.check(L.pgmoe_gather_rows(_ptr(x), _ptr(r_in.perm), n, d, k, _ptr(x_send), _stream(stream)))
        x_recv = self.ex.rows(x_send[:n], send_splits, recv_splits)
        n_recv = x_recv.shape[0]
        if n_recv > self.max_recv:
            raise ShapeError("received more rows than the EP buffers hold")
        _lib.check(L.pgmoe_ep_local_routing(_ptr(recv_cnt), self.P, self.El, ctypes.byref(self.lr.c),
                                            _stream(stream)))
        base, stride = ctypes.c_void_p(), ctypes.c_size_t()
        eb, nl = ctypes.c_int32(), ctypes.c_int32()
        _lib.check(L.pgmoe_model_expert_records(self.model._h, b, ctypes.byref(base), ctypes.byref(stride),
                                                ctypes.byref(eb), ctypes.byref(nl)))
        h = torch.empty((max(n_recv, 1), f), dtype=torch.float32, device=x.device)
        y_recv = torch.empty((max(n_recv, 1), d), dtype=torch.float32, device=x.device)
        if n_recv:
            from .core import _KERNEL
            _lib.check(L.pgmoe_expert_forward(_ptr(x_recv), n_recv, d, f, 1, base, stride.value,
                                              self.model.wdt, 0, ctypes.byref(self.lr.c), _ptr(h), _ptr(y_recv),
                                              _KERNEL[self.kernel], _stream(stream)))
        back = self.ex.rows(y_recv[:n_recv], recv_splits, send_splits)
        yw = torch.empty((max(n, 1), d), dtype=torch.float32, device=x.device)
        _lib.check(L.pgmoe_unpermute_combine(_ptr(back), _ptr(r_in.perm), _ptr(r_in.w_perm), n, d, _ptr(yw),
                                             _stream(stream)))
        y = torch.empty_like(x)
        from .core import _KERNEL
        _lib.check(L.pgmoe_dense_forward(_ptr(yw), T, d, k, _ptr(self.model.matrix("non_moe", b)),
                                         self.model.wdt, _ptr(y), _KERNEL[self.kernel], _stream(stream)))
        return y

    def decoder_iteration(self, x: torch.Tensor, trace: bool = False):
        """Local tokens x [T][d] (cuda fp32) -> (y, consumed ids per block).

        With the fixed-size exchange nothing in an iteration waits on the
        host, so the whole iteration (routing, packs, NCCL all-to-alls, FFN,
        combine, dense) is captured once per input buffer into a CUDA graph
        and replayed; the returned y is the graph's output buffer."""
        if self.packed and self.use_graph and not trace:
            key = (x.data_ptr(), tuple(x.shape))
            entry = self._graphs.get(key)
            if entry is None:
                # a capture failure is an error, not a silent switch to eager
                # execution (PGMOE_EP_GRAPH=0 selects eager launches explicitly)
                try:
                    entry = self._capture(x)
                except Exception as e:  # noqa: BLE001
                    raise DeviceError(f"EP CUDA-graph capture failed: {e} (set PGMOE_EP_GRAPH=0 for eager "
                                      "launches)") from e
                if len(self._graphs) >= 4:
                    self._graphs.pop(next(iter(self._graphs)))
                self._graphs[key] = entry
            g, y, n = entry
            g.replay()
            self.replayed_kernels += n
            return y, None
        return self._iteration(x, trace)

    def _capture(self, x: torch.Tensor):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._iteration(x, False)  # warm-up: communicators, workspaces, allocator
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = self._L.pgmoe_launch_count()
        with torch.cuda.graph(g):
            y, _ = self._iteration(x, False)
        return g, y, self._L.pgmoe_launch_count() - n0  # our kernels per replay

    def _rbuf(self, T: int, slot: int) -> DeviceRouting:
        """Routing buffers reused across blocks and iterations (a fresh
        DeviceRouting zero-fills nine tensors: nine extra launches per block)."""
        key = (T, slot)
        r = self._rbufs.get(key)
        if r is None:
            r = self._rbufs[key] = DeviceRouting(T, self.config.num_experts, self.config.top_k)
        return r

    def _iteration(self, x: torch.Tensor, trace: bool = False):
        """The decoder loop (core.py:342-383).  Pre-gating at work: block b's
        pre-gate reads only block b's input, so it runs on a side stream
        concurrently with block b's exchange and expert FFN and is off the
        critical path (the consumer waits on its event one block later)."""
        from .core import route
        c = self.config
        main = torch.cuda.current_stream()
        pending: dict = {}
        ids = []
        T = x.shape[0]
        for b in range(c.num_blocks):
            if c.has_conv_gate(b):
                r_in = route(x, self.model.matrix("gate", b), c.top_k, out=self._rbuf(T, 2))
            else:
                r_in, done = pending.pop(b)
                main.wait_event(done)
            if c.has_pre_gate(b):
                ready = torch.cuda.Event()
                ready.record(main)  # block b's input is written (and block b-1 is done with its routing)
                self._side.wait_event(ready)
                with torch.cuda.stream(self._side):
                    r = route(x, self.model.matrix("pre_gate", b), c.top_k,
                              out=self._rbuf(T, (b + c.activation_level) % (c.activation_level + 1)))
                    done = torch.cuda.Event()
                    done.record(self._side)
                x.record_stream(self._side)
                pending[b + c.activation_level] = (r, done)
            if trace:
                ids.append(r_in.ids.clone())
            x = self.block(b, x, r_in)
        return x, (torch.stack(ids) if trace else None)

    def close(self):
        self.model.close()
