"""TEST INFRASTRUCTURE ONLY — parity measurements of a GPU decoder run
against the oracle (tests/ and bench.py's after-the-timed-region check).

Two measurements, both on the reference's arithmetic (oracle/pgmoe_oracle.c,
pinned bit-for-bit to moesim by tests/test_oracle.py):

* ``teacher_forced`` — SURVEY §8(c): every block of a GPU iteration is
  re-run by the oracle on the GPU's OWN block input (x_trace[b], promoted to
  fp64).  Routing ids of ALL tokens at every block must equal the oracle's
  (the consumed decision of block b is the oracle's gate on the GPU's input
  of block b - L, core.py:342-383 wiring); block outputs of sampled tokens
  are compared normwise (||y - y_ref||_inf / ||y_ref||_inf per token).
* ``chained`` — the GPU's own chain next to the oracle's fp64 chain
  (core.py:342-383 with x_{it+1} = y_it, scheduler.py:252-255) on sampled
  tokens: routing flips per block (ids that differ from the reference's)
  and the normwise divergence per block.  Nothing is teacher-forced, so a
  flip propagates; the first flip of every token is reported.

The reference's synthetic model has no residual or normalisation, so the
activation magnitude decays ~14x per block (Switch-Large dims, measured);
fp32 (the GPU's inter-block storage) leaves its normal range after
~1.3 decoder iterations while fp64 lasts ~10.  Blocks whose GPU input is
below FP32_NORMAL_MIN are reported separately ("underflowed").
"""

from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np

from . import oracle as og

FP32_NORMAL_MIN = float(np.finfo(np.float32).tiny)  # 1.18e-38


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _materialize(model: og.OracleModel, b: int, experts, nthreads: int) -> None:
    """Generate (in parallel: ctypes releases the GIL) the expert matrices of
    block b that the next oracle call needs."""
    todo = [e for e in sorted(set(int(e) for e in experts)) if ("w1", b, e) not in model._cache]
    if not todo:
        return
    with cf.ThreadPoolExecutor(max_workers=nthreads) as ex:
        list(ex.map(lambda e: (model.w1(b, e), model.w2(b, e)), todo))


def _drop_block(model: og.OracleModel, b: int) -> None:
    for key in [k for k in model._cache if k[1] == b and k[0] in ("w1", "w2")]:
        del model._cache[key]


def _decision_gate(dims: og.Dims, model: og.OracleModel, b: int):
    """(gate matrix, block whose input it reads) of block b's consumed decision."""
    if dims.has_conv_gate(b):
        return model.gate(b), b
    src = b - dims.activation_level
    return model.pre_gate(src), src


def normwise_rows(y: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """||y_t - ref_t||_inf / ||ref_t||_inf per row t."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref), axis=1)
    num = np.max(np.abs(y - ref), axis=1)
    return num / np.where(den > 0, den, 1.0)


def teacher_forced(dims: og.Dims, dtype: str, x_trace: np.ndarray, y: np.ndarray, ids_trace: np.ndarray,
                   w_trace: np.ndarray, sample: np.ndarray, blocks, nthreads: int = 0,
                   model: og.OracleModel | None = None) -> dict:
    """Check one GPU decoder iteration (x_trace [nb][T][d], y [T][d],
    ids_trace / w_trace [nb][T][k]) block by block against the oracle.

    ids: every token, every block whose decision-source input is in the
    fp32 normal range.  Outputs: tokens `sample`, blocks `blocks`."""
    nthreads = nthreads or _threads()
    model = model or og.OracleModel(dims, dtype)
    nb, T, d = x_trace.shape
    k = dims.top_k
    out = {"blocks": [], "ids_blocks_checked": 0, "ids_mismatch_tokens": 0, "w_max_rel": 0.0,
           "max_err": 0.0, "tokens": int(len(sample)), "underflowed_blocks": []}
    for b in range(nb):
        G, src = _decision_gate(dims, model, b)
        xs = x_trace[src].astype(np.float64)
        if np.max(np.abs(xs)) < FP32_NORMAL_MIN:
            out["underflowed_blocks"].append(b)
            continue
        ids_ref, w_ref = og.gate_batch(xs, G, k, nthreads)
        mism = int(np.sum(np.any(ids_ref != ids_trace[b], axis=1)))
        out["ids_blocks_checked"] += 1
        out["ids_mismatch_tokens"] += mism
        if mism == 0:
            rel = np.abs(w_trace[b].astype(np.float64) - w_ref) / w_ref
            out["w_max_rel"] = max(out["w_max_rel"], float(np.max(rel)))
        if b not in blocks:
            continue
        xb = x_trace[b][sample].astype(np.float64)
        if np.max(np.abs(xb)) < FP32_NORMAL_MIN:
            out["underflowed_blocks"].append(b)
            continue
        ids_s, w_s = ids_ref[sample], w_ref[sample]
        _materialize(model, b, ids_s.reshape(-1), nthreads)
        w1 = {int(e): model.w1(b, int(e)) for e in np.unique(ids_s)}
        w2 = {int(e): model.w2(b, int(e)) for e in np.unique(ids_s)}
        y_ref = og.block_batch(xb, ids_s, w_s, w1, w2, model.dense(b), dims.num_experts, nthreads)
        y_gpu = (x_trace[b + 1] if b + 1 < nb else y)[sample]
        err = float(np.max(normwise_rows(y_gpu, y_ref)))
        out["blocks"].append({"block": b, "err": err, "ids_equal": mism == 0})
        out["max_err"] = max(out["max_err"], err)
        _drop_block(model, b)
    return out


def chained(dims: og.Dims, dtype: str, x0: np.ndarray, gpu_x: list, gpu_ids: list, nthreads: int = 0,
            model: og.OracleModel | None = None) -> dict:
    """The oracle's fp64 chain from the sampled fp32 tokens x0 [S][d] over
    len(gpu_x) decoder iterations, beside the GPU's chain: gpu_x[it] =
    block inputs [nb][S][d] of iteration it (gpu_x[it+1][0] = GPU output
    of iteration it), gpu_ids[it] = consumed ids [nb][S][k].  Returns per
    (iteration, block): flips (tokens whose ids differ from the
    reference's), normwise divergence of the block input, and whether the
    GPU's input had left the fp32 normal range."""
    nthreads = nthreads or _threads()
    model = model or og.OracleModel(dims, dtype)
    k = dims.top_k
    x = np.asarray(x0, dtype=np.float64)
    S = x.shape[0]
    rows = []
    first_flip = [None] * S
    for it, (gx, gi) in enumerate(zip(gpu_x, gpu_ids)):
        pending: dict = {}
        for b in range(dims.num_blocks):
            err = float(np.max(normwise_rows(gx[b], x)))
            under = bool(np.max(np.abs(gx[b])) < FP32_NORMAL_MIN)
            if dims.has_conv_gate(b):
                ids, w = og.gate_batch(x, model.gate(b), k, nthreads)
            else:
                ids, w = pending.pop(b)
            if dims.has_pre_gate(b):
                pending[b + dims.activation_level] = og.gate_batch(x, model.pre_gate(b), k, nthreads)
            diff = np.any(ids != gi[b], axis=1)
            for t in np.nonzero(diff)[0]:
                if first_flip[t] is None:
                    first_flip[t] = [it, b]
            rows.append({"iteration": it, "block": b, "flips": int(diff.sum()), "input_err": err,
                         "gpu_input_underflowed": under})
            _materialize(model, b, ids.reshape(-1), nthreads)
            w1 = {int(e): model.w1(b, int(e)) for e in np.unique(ids)}
            w2 = {int(e): model.w2(b, int(e)) for e in np.unique(ids)}
            x = og.block_batch(x, ids, w, w1, w2, model.dense(b), dims.num_experts, nthreads)
            _drop_block(model, b)
    in_range = [r for r in rows if not r["gpu_input_underflowed"]]
    return {
        "tokens": S,
        "iterations": len(gpu_x),
        "flips_total": int(sum(r["flips"] for r in rows)),
        "flips_in_fp32_range": int(sum(r["flips"] for r in in_range)),
        "token_blocks_in_fp32_range": len(in_range) * S,
        "first_underflow": next(([r["iteration"], r["block"]] for r in rows if r["gpu_input_underflowed"]), None),
        "first_flip": first_flip,
        "per_block": rows,
    }
