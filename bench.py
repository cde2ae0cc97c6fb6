"""Benchmark of the B200 pre-gated MoE block (contract: one JSON line on rank 0).

Workload (BASELINE.json metric "MoE tokens/sec & per-block latency (1 GPU
offloaded; 2/4/8 EP)"): configs[3] Switch-Large-128 (d=1024, f=4096, E=128,
top-1, 24 blocks, activation level 1), bf16 weights, experts offloaded to
pinned host memory with pre-gated prefetch into a 2-slot HBM expert cache.
A step = one decoder iteration (core.py:342-383) over a batch of T synthetic
tokens (SURVEY §8(d) token recipe).  Each step's expert traffic (~45 GB at
T=256) is far larger than L2, so no explicit flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--tokens T]
                    [--impl ours|reference] [--preset large128|base128|base64]
                    [--placement offloaded|resident]

--impl reference times the reference's CPU implementation of the path (the
oracle's C restatement of moesim, all host threads) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PRESETS = {  # presets.py:64-70 full-size dims
    "base8": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=8),
    "base64": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=64),
    "base128": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=128),
    "large128": dict(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128),
}
METRIC = "MoE tokens/sec & per-block latency (1 GPU offloaded; 2/4/8 EP) vs CPU ref; % roofline"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~0.1-0.5 s for its first line: wait for it, so
            # a timed region shorter than the sampling period still has the
            # sample taken at its start
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measure_pcie_gbs(torch, nbytes=1 << 30, reps: int = 3) -> float:
    """Pinned host -> device copy bandwidth: best of `reps` timings of four
    back-to-back 1 GiB copies (a peak, like MEASURED_PEAKS.json's best-of-10;
    one timing measured up to ~1 % low on some boxes)."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(4):
            d.copy_(h, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, 4 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    del h, d
    return best


PEAK_NOTE = ("peak: MEASURED_PEAKS.json hbm_gbs, a device-to-device copy (read + write bytes); a read-only weight "
             "stream can exceed it slightly")


def workload_name(preset: str, placement: str, tokens: int) -> str:
    """BASELINE.json configs index of a single-GPU workload."""
    idx = {("base8", "offloaded"): 0, ("base8", "resident"): 0, ("base64", "resident"): 1,
           ("base128", "offloaded"): 2, ("large128", "offloaded"): 3}.get((preset, placement))
    tag = f" (BASELINE configs[{idx}])" if idx is not None else ""
    return f"Switch-{preset} {placement} pre-gated T={tokens}{tag}"


def ncu_traffic(kernel_label: str, workload: str):
    """Per-launch DRAM bytes (read + write) of the dominant kernel from the
    committed ncu summary of THIS workload (profiles/*ncu_summary*.json
    carrying the same `workload`), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu_summary*.json")), reverse=True):
        try:
            with open(path) as fh:
                s = json.load(fh)
            if s.get("workload") != workload:
                continue
            k = s.get("kernels", {}).get(kernel_label)
            if k and k.get("dram_bytes_per_launch"):
                return k["dram_bytes_per_launch"]
        except Exception:
            continue
    return None


# ------------------------------------------------------------ CPU side ----

def cpu_reference_run(preset: str, dtype: str, T_sample: int, steps: int, warmup: int, nthreads: int,
                      seed: int = 0):
    """The reference algorithm (oracle = C restatement of moesim, validated
    bit-exact against moesim) on T_sample tokens, one decoder iteration per
    step (the same fresh synthetic batch every step, like our arm).  Weights
    are materialised in parallel before each block and excluded from timing
    (as in the reference's own measurements); they stay cached (warm) when
    host RAM allows, else they are regenerated per block."""
    import numpy as np
    from oracle import oracle as og
    from oracle.parity import _drop_block, _materialize
    from paper_2308_12066_b200._rng import token_batch

    p = PRESETS[preset]
    dims = og.Dims(p["d_model"], p["d_ff"], p["num_blocks"], p["num_experts"], 1, 1, seed)
    model = og.OracleModel(dims, dtype)
    x0 = token_batch(seed, dims.d_model, T_sample).astype(np.float64)
    rec = 2 * dims.d_model * dims.d_ff * (2 if dtype == "bf16" else 4)
    n_act = dims.num_experts * (1 - (1 - 1 / dims.num_experts) ** T_sample)
    need = dims.num_blocks * n_act * rec
    try:
        import psutil
        keep = psutil.virtual_memory().available > 2.5 * need
    except Exception:
        keep = False

    def one_iteration() -> float:
        x = x0
        spent = 0.0
        pending = {}
        for b in range(dims.num_blocks):
            G = model.gate(b) if dims.has_conv_gate(b) else None
            PG = model.pre_gate(b) if dims.has_pre_gate(b) else None
            D = model.dense(b)
            t = time.perf_counter()
            if G is not None:
                ids, w = og.gate_batch(x, G, 1, nthreads)
            else:
                ids, w = pending.pop(b)
            if PG is not None:
                pending[b + 1] = og.gate_batch(x, PG, 1, nthreads)
            spent += time.perf_counter() - t
            _materialize(model, b, ids.reshape(-1), nthreads)  # untimed
            w1 = {int(e): model.w1(b, int(e)) for e in np.unique(ids)}
            w2 = {int(e): model.w2(b, int(e)) for e in np.unique(ids)}
            t = time.perf_counter()
            x = og.block_batch(x, ids, w, w1, w2, D, dims.num_experts, nthreads)
            spent += time.perf_counter() - t
            if not keep:
                _drop_block(model, b)
        return spent

    for _ in range(warmup):
        one_iteration()
    return [one_iteration() for _ in range(steps)]


# ------------------------------------------------------------- GPU side ----

def block_latencies(events: list, nb: int) -> list:
    """Per-block latencies of consecutive decoder iterations from a timeline:
    a block's latency is the time between the ends of consecutive blocks'
    dense layers (scheduler.py:374-379), block 0 measured from the start of
    its iteration.  Returns [iterations][nb]."""
    dense = [e for e in events if e["label"] == "non_moe"]
    out, prev = [], None
    starts = sorted(e["start_s"] for e in events)
    t0 = starts[0] if starts else 0.0
    for i, e in enumerate(dense):
        if i % nb == 0:
            out.append([])
            prev = t0 if i == 0 else prev
        out[-1].append(e["end_s"] - prev)
        prev = e["end_s"]
    return out


def run_parity(model, x, dims, dtype: str, sample_n: int, chained_n: int, chained_iters: int) -> tuple:
    """After the timed region: the bench's own model and launch sequence,
    checked against the oracle (oracle/parity.py) — teacher-forced on every
    block (ids of all T tokens, outputs of `sample_n` sampled tokens at 4
    blocks incl. the last) and the chained flip measurement (`chained_n`
    tokens, `chained_iters` chained iterations, no teacher forcing)."""
    import numpy as np
    import torch
    from oracle import oracle as og
    from oracle import parity

    c = model.config
    T = x.shape[0]
    nb = c.num_blocks
    xt = torch.empty((nb, T, c.d_model), dtype=torch.float32, device="cuda")
    ids = torch.empty((nb, T, c.top_k), dtype=torch.int32, device="cuda")
    w = torch.empty((nb, T, c.top_k), dtype=torch.float32, device="cuda")
    y_plain, y_tr = torch.empty_like(x), torch.empty_like(x)
    runs, cur = [], x
    for it in range(max(1, chained_iters)):
        model.decoder_iteration(cur, out=y_plain)
        model.decoder_iteration(cur, out=y_tr, x_trace=xt, trace_out=(ids, w))
        torch.cuda.synchronize()
        model.check_routing()
        same = bool(torch.equal(y_plain, y_tr))
        runs.append((xt.cpu().numpy(), y_tr.cpu().numpy(), ids.cpu().numpy(), w.cpu().numpy(), same))
        cur = y_tr.clone()
    om = og.OracleModel(og.Dims(c.d_model, c.d_ff, nb, c.num_experts, c.top_k, c.activation_level, c.seed), dtype)
    sample = np.linspace(0, T - 1, sample_n).astype(int)
    xt0, y0, ids0, w0, same0 = runs[0]
    tf = parity.teacher_forced(dims, dtype, xt0, y0, ids0, w0, sample, {0, 1, nb // 2, nb - 1}, model=om)
    par = {"method": "teacher-forced per block on the timed path's own block inputs (oracle/parity.py)",
           "traced_equals_plain": same0, "ids_tokens_x_blocks": tf["ids_blocks_checked"] * T,
           "ids_mismatch_tokens": tf["ids_mismatch_tokens"], "w_max_rel": tf["w_max_rel"],
           "sampled_tokens": len(sample), "blocks": [[b["block"], round(b["err"], 6)] for b in tf["blocks"]],
           "max_err": tf["max_err"], "tol": 2e-2 if dtype == "bf16" else 1e-4}
    par["pass"] = bool(same0 and tf["ids_mismatch_tokens"] == 0 and tf["max_err"] <= par["tol"])
    chained = None
    if chained_iters > 0:
        cs = np.linspace(0, T - 1, chained_n).astype(int)
        ch = parity.chained(dims, dtype, runs[0][0][0][cs], [r[0][:, cs] for r in runs],
                            [r[2][:, cs] for r in runs], model=om)
        first = [f for f in ch["first_flip"] if f is not None]
        chained = {"tokens": ch["tokens"], "iterations": ch["iterations"], "flips_total": ch["flips_total"],
                   "flips_in_fp32_range": ch["flips_in_fp32_range"],
                   "token_blocks_in_fp32_range": ch["token_blocks_in_fp32_range"],
                   "first_flip_per_token": ch["first_flip"],
                   "first_gpu_fp32_underflow": ch["first_underflow"],
                   "flips_per_block": [r["flips"] for r in ch["per_block"]],
                   "input_err_per_block": [float("%.3g" % r["input_err"]) for r in ch["per_block"]],
                   "note": "GPU bf16/fp32 chain vs the oracle's fp64 chain (x_{it+1} = y_it, scheduler.py:252-255), "
                           "no teacher forcing; a flip diverges that token's trajectory"}
        if first:
            chained["earliest_flip"] = min(first)
    return par, chained


def run_ours(args, rank: int, world: int):
    import numpy as np
    import torch
    import paper_2308_12066_b200 as P
    from paper_2308_12066_b200 import _lib
    from paper_2308_12066_b200._rng import token_batch

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    pr = PRESETS[args.preset]
    cfg = P.ModelConfig(top_k=1, activation_level=1, seed=0, **pr)
    T = args.tokens
    t_setup = time.perf_counter()
    model = P.DeviceModel(cfg, dtype=args.dtype, placement=args.placement, max_tokens=T, kernel=args.kernel)
    setup_s = time.perf_counter() - t_setup
    # each rank owns its own T sequences (weak scaling over sequences)
    x_host = torch.from_numpy(token_batch(0, cfg.d_model, T, offset=rank * T)).pin_memory()
    x = x_host.cuda()
    stream = torch.cuda.current_stream()
    L = _lib.load()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    y_buf = torch.empty_like(x)
    for _ in range(args.warmup):
        model.decoder_iteration(x, out=y_buf)
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs (resident: CUDA-graph replay) --
    model.reset_stats()
    launches0 = L.pgmoe_launch_count()
    clocks = ClockSampler(dev)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        model.decoder_iteration(x, out=y_buf)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = L.pgmoe_launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    st = model.stats()
    model.check_routing()
    # the reference's steady block latency (scheduler.py:374-397: between consecutive dense-layer
    # ends, blocks 1..nb-1) from device stamps the chained block launches write in the timed,
    # graph-replayed iterations themselves (read before the profile pass overwrites them)
    stamps = np.zeros(cfg.num_blocks + 1, dtype=np.int64)
    _lib.check(L.pgmoe_model_block_stamps(model._h, stamps.ctypes.data, cfg.num_blocks + 1))
    st_ms = np.diff(stamps[1:]) / 1e6
    steady_stamped_ms = float(st_ms.mean()) if (stamps[1:] > 0).all() and (st_ms > 0).all() else None
    # ---- profile pass: per-kernel CUDA events on the compute / copy streams
    prof_steps = max(1, min(args.steps, 3))
    model.set_timeline(True)
    ll0, dec0 = model.ll_decode_iterations, model.decode_iterations
    for _ in range(prof_steps):
        model.decoder_iteration(x)
    torch.cuda.synchronize()
    # which launch served the iteration: the low-latency decoder (decode_ll.cu), the
    # persistent tcgen05 decoder (decode_tc.cu) or one block launch per block (ffn_tc.cu)
    served = ("ll" if model.ll_decode_iterations > ll0 else "decode" if model.decode_iterations > dec0 else "blocks")
    tl = model.timeline()
    model.set_timeline(False)
    # the profile pass runs the host loop (no graph replay), so its stats say
    # which stages ran inside the block launch
    st_prof = model.stats()
    gpu_launches_per_step = launches / args.steps

    # ---- per-kernel roofline from the CUDA events on the compute stream ---
    hbm_peak, tc_peak, peak_kind = peaks()
    sw = 2 if args.dtype == "bf16" else 4
    d, f, E, nb = cfg.d_model, cfg.d_ff, cfg.num_experts, cfg.num_blocks
    rec = 2 * d * f * sw
    ffn = [e for e in tl if e["label"] == "experts"]
    ffn_s = sum(e["end_s"] - e["start_s"] for e in ffn)
    # measured n_act per block from the transfer labels "fetch[n]" (offloaded)
    fetch = [e for e in tl if e["lane"] == "transfer"]
    if fetch:
        nact_total = sum(int(e["label"][6:-1]) for e in fetch)
    else:  # resident: recompute from one traced iteration
        _, ids, _ = model.decoder_iteration(x, trace=True)
        torch.cuda.synchronize()
        nact_total = sum(len(torch.unique(ids[b])) for b in range(nb)) * prof_steps
    # per routed token: bf16 x packed+read, bf16 h write+read, fp32 yw + bf16 mix written
    act_bytes_per_token = 2 * d * 2 + 2 * f * 2 + d * 6
    ffn_bytes = nact_total * rec + prof_steps * nb * T * act_bytes_per_token
    fused = st_prof.get("fused_blocks", 0) > 0
    if fused:  # the dense layer runs inside the same launch: its weights and activations
        ffn_bytes += prof_steps * nb * (d * d * sw + T * d * (2 + 4))
    routed_in_launch = st_prof.get("fused_routes", 0) > 0
    if routed_in_launch:  # resident: the next block's pre-gate (gate weights + block input) too
        ffn_bytes += prof_steps * (nb - 1) * (d * E * sw + T * d * 4)
    ffn_gbs = ffn_bytes / ffn_s / 1e9 if ffn_s > 0 else None
    h2d_s = sum(e["end_s"] - e["start_s"] for e in fetch)
    pcie_gbs = measure_pcie_gbs(torch)
    h2d_gbs = (nact_total * rec / h2d_s / 1e9) if (h2d_s > 0 and fetch) else None
    # per-block roofline time: max(HBM, tensor, PCIe)
    nact_avg = nact_total / (prof_steps * nb)
    n_gates_avg = cfg.gate_count / nb
    hbm_b = n_gates_avg * d * E * sw + nact_avg * rec + d * d * sw + T * d * 4 * 5 + T * 8 + (2 * E + 1) * 4
    flops = n_gates_avg * 2 * T * d * E + 4 * T * d * f + 2 * T * d * d
    pcie_b = nact_avg * rec if args.placement == "offloaded" else 0
    bounds = {"hbm": hbm_b / (hbm_peak * 1e9), "tensor": flops / (tc_peak * 1e12),
              "pcie": pcie_b / (pcie_gbs * 1e9)}
    bound = max(bounds, key=bounds.get)
    t_roof = bounds[bound]
    phases = {}
    for e in tl:
        key = e["lane"] + ":" + e["label"].split("[")[0]
        phases[key] = phases.get(key, 0.0) + (e["end_s"] - e["start_s"])
    phases = {k: round(v * 1e3 / (prof_steps * nb), 4) for k, v in phases.items()}
    # the reference's metric definitions (scheduler.py:387-407): block
    # latency = time between consecutive blocks' dense-layer ends, averaged
    # over blocks 1..nb-1 (block 0 — the exposed serial fetch — apart)
    lats = block_latencies(tl, nb)
    steady = [v for it in lats for v in it[1:]]
    block0 = [it[0] for it in lats]
    per_block_ms = statistics.mean(steady) * 1e3 if steady else ms / nb
    per_block_src = "profile-pass CUDA events" if steady else "timed ms_per_step / num_blocks (one launch per iteration)"
    if steady_stamped_ms is not None and args.placement == "resident":
        # chained resident launches: per-launch events would serialise them; the device stamps don't
        per_block_ms, per_block_src = steady_stamped_ms, "device dense-end stamps of the timed iterations"
    block0_ms = statistics.mean(block0) * 1e3 if block0 else None
    # steady_state_latency closed form (scheduler.py:180-196), pre_gated:
    # max(block compute, transfer of the routed experts), from measured parts
    compute_ms = sum(v for k, v in phases.items() if k.startswith("compute:") and k != "compute:gate")
    transfer_ms = pcie_b / (pcie_gbs * 1e9) * 1e3
    closed_ms = max(compute_ms, transfer_ms) if args.placement == "offloaded" else compute_ms

    # ---- end to end through the C ABI with host buffers, every step -----
    y_host = torch.empty_like(x_host).pin_memory()
    # one untimed call: the host entry point's device buffers (and, resident,
    # its CUDA graph) are created on first use
    _lib.check(L.pgmoe_decoder_iteration_host(model._h, _ptr(x_host), T, _ptr(y_host), None, None))
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _lib.check(L.pgmoe_decoder_iteration_host(model._h, _ptr(x_host), T, _ptr(y_host), None, None))
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- chaining y -> x across steps (diagnostic, not the headline) -----
    # The synthetic model has no residual/normalisation: activations decay
    # ~14x per block, so a chained fp32 batch leaves the normal range after
    # ~1.3 iterations and every later block routes all-zero inputs to expert
    # 0 (n_act -> 1): a degenerate, far cheaper workload.  Measured here so the
    # headline's fresh-batch choice is evidenced, not asserted.
    chain_diag = None
    if rank == 0 and not args.no_parity:
        cur = x.clone()
        nxt = torch.empty_like(x)
        per_it = []
        for _ in range(4):
            a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            _, ids_c, _ = model.decoder_iteration(cur, out=nxt, trace=True)
            b2.record(stream)
            torch.cuda.synchronize()
            nact = [len(torch.unique(ids_c[bb])) for bb in range(nb)]
            per_it.append({"ms": round(a.elapsed_time(b2), 3), "n_act_avg": round(sum(nact) / nb, 2),
                           "max_abs_input": float("%.3g" % cur.abs().max().item())})
            cur, nxt = nxt, cur
        chain_diag = {"iterations": per_it,
                      "note": "x_{it+1} = y_it; n_act collapses once fp32 activations underflow, so the headline "
                              "times a fresh synthetic batch every step (same routing statistics as the "
                              "reference's fp64 chain, whose ranking is scale-invariant)"}

    # ---- parity of the timed path (rank 0): oracle on the bench's shapes --
    par = chained = None
    if rank == 0 and not args.no_parity:
        from oracle import oracle as og
        dims = og.Dims(d, f, nb, E, 1, 1, 0)
        par, chained = run_parity(model, x, dims, args.dtype, 8, 4, 3)

    out = {
        "metric": METRIC,
        "value": round(T * world / (ms * 1e-3), 3),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (reference RNG weights/tokens, SURVEY §8(d))",
        "config": {"workload": workload_name(args.preset, args.placement, T) +
                               (" f32 weights" if args.dtype == "f32" else ""),
                   "preset": args.preset, "placement": args.placement, "tokens_per_rank": T,
                   "global_batch": T * world, "num_blocks": nb, "d_model": d, "d_ff": f, "num_experts": E,
                   "top_k": 1, "activation_level": 1, "parallelism": f"sequences x{world} (replicas)",
                   "inputs": "the same fresh synthetic batch every step (see chained_steps)",
                   "l2": "inputs larger than L2: per-step expert bytes >> 126 MB (streamed evict-first); only the "
                         "dense weights (d^2 per block, loaded evict-last) may stay L2-resident across steps",
                   "kernel": args.kernel},
        "per_block_latency_ms": round(per_block_ms, 4),
        "block0_latency_ms": round(block0_ms, 4) if block0_ms is not None else None,
        "per_block_latency_all_blocks_ms": round(ms / nb, 4),
        "per_block_latency_source": per_block_src,
        "latency_note": "per_block_latency_ms / block0_latency_ms: the reference's definition (scheduler.py:374-397: "
                        "ends of consecutive dense layers, block 0 excluded from the average); see "
                        "per_block_latency_source; per_block_latency_all_blocks_ms = timed ms_per_step / num_blocks",
        "steady_state_closed_form_ms": round(closed_ms, 4),
        "steady_state_measured_over_closed_form": round(per_block_ms / closed_ms, 4) if closed_ms else None,
        "per_block_phase_ms": phases,
        "block_roofline": {"t_roof_ms": round(t_roof * 1e3, 4), "frac": round(t_roof * 1e3 / per_block_ms, 4),
                           "bound": bound,
                           "peak_note": ("hbm peak = MEASURED_PEAKS hbm_gbs, a device copy (read + write); the "
                                         "block's traffic is almost all weight reads, which can stream faster, so "
                                         "frac may exceed 1") if bound == "hbm" else
                                        ("pcie peak = best of 3 timings of 4 x 1 GiB pinned H2D copies in this "
                                         "process" if bound == "pcie" else None),
                           "t_hbm_ms": round(bounds["hbm"] * 1e3, 4),
                           "t_tensor_ms": round(bounds["tensor"] * 1e3, 4),
                           "t_pcie_ms": round(bounds["pcie"] * 1e3, 4), "n_act_avg": round(nact_avg, 2)},
        "roofline": {"bound": "hbm",
                     "kernel": ({"ll": "ll_decode_kernel (decode_ll.cu): every block's up+down+dense and pre-gates, "
                                       "one launch per decoder iteration",
                                 "decode": "decode_kernel (decode_tc.cu): every block, one launch per iteration"}
                                .get(served) or ("K2 up+down" + (" + K3 dense" if fused else "") +
                                                 (" + next block's K1 routing" if routed_in_launch else "") +
                                                 (", one launch" if fused else ""))),
                     "achieved": round(ffn_gbs, 1) if ffn_gbs else None, "peak": hbm_peak,
                     "unit": "GB/s", "frac": round(ffn_gbs / hbm_peak, 4) if ffn_gbs else None,
                     "traffic": ncu_traffic("ffn", workload_name(args.preset, args.placement, T) +
                                            (" f32 weights" if args.dtype == "f32" else "")),
                     "peak_kind": peak_kind, "peak_note": PEAK_NOTE if peak_kind == "measured" else None,
                     "algorithmic_bytes_per_launch": round(ffn_bytes / max(1, len(ffn))),
                     "avg_launch_us": round(ffn_s / max(1, len(ffn)) * 1e6, 2)},
        "migration": {"h2d_gbs": round(h2d_gbs, 2) if h2d_gbs else None, "pcie_measured_gbs": round(pcie_gbs, 2),
                      "frac": round(h2d_gbs / pcie_gbs, 4) if h2d_gbs else None,
                      "h2d_bytes_per_step": st["h2d_bytes"] // max(1, args.steps),
                      "copy_busy_frac": round(h2d_s / (ms * 1e-3 * prof_steps), 4) if h2d_s else None,
                      "peak_hbm_eq1_bytes": st["eq1_peak_bytes"], "peak_hbm_ledger_bytes": st["ledger_peak_bytes"],
                      "pinned_hbm_bytes": st["pinned_hbm_bytes"]},
        "routing": {"serial_fallbacks": st["route_fallbacks"], "chained": chained},
        "parity": par,
        "chained_steps": chain_diag,
        "e2e": {"value": round(T * world / e2e_s, 3), "unit": "tokens/s",
                "h2d_bytes_per_step": T * d * 4, "d2h_bytes_per_step": T * d * 4, "steps": args.steps},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": gpu_launches_per_step,
        "clocks": clk,
        "setup_s": round(setup_s, 2),
        "timing_note": "value/ms_per_step: CUDA events around the K timed steps (resident: CUDA-graph replay); "
                       "roofline/phases/per-block latencies: a following pass with per-kernel CUDA events on the "
                       "same streams; e2e: host wall clock over K steps through pgmoe_decoder_iteration_host",
    }
    # ---- CPU baseline (rank 0, N=1 only): the same workload, all T tokens -
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        sample = args.cpu_sample or T
        t_cpu = time.perf_counter()
        times = cpu_reference_run(args.preset, args.dtype, sample, 2, 1, nth)  # one untimed warm-up iteration
        out["cpu_baseline"] = {"value": round(sample / statistics.mean(times), 4), "unit": "tokens/s",
                               "cores": nth, "kind": "port",
                               "sample": f"{sample} tokens x 1 decoder iteration ({nb} blocks) per step, 2 timed "
                                         f"after 1 warm-up, oracle C restatement of moesim, {nth} threads "
                                         f"({time.perf_counter() - t_cpu:.0f} s wall incl. weight generation)"}
    model.close()
    return out


def _ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def run_ep(args, rank: int, world: int):
    """configs[4]: Switch-Large-128 expert-parallel over `world` GPUs (experts
    sharded, resident in HBM), NCCL all-to-all dispatch/combine, T tokens
    per rank (weak scaling)."""
    import torch
    import paper_2308_12066_b200 as P
    from paper_2308_12066_b200 import _lib
    from paper_2308_12066_b200._rng import token_batch
    from paper_2308_12066_b200.ep import EPDecoder

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    pr = PRESETS[args.preset]
    cfg = P.ModelConfig(top_k=1, activation_level=1, seed=0, **pr)
    T = args.tokens
    t_setup = time.perf_counter()
    dec = EPDecoder(cfg, dtype="bf16", max_tokens=T, kernel=args.kernel)
    setup_s = time.perf_counter() - t_setup
    x_host = torch.from_numpy(token_batch(0, cfg.d_model, T, offset=rank * T)).pin_memory()
    x = x_host.cuda()
    L = _lib.load()
    for _ in range(args.warmup):
        dec.decoder_iteration(x)
    torch.cuda.synchronize()
    launches0 = L.pgmoe_launch_count() + dec.replayed_kernels
    clocks = ClockSampler(dev)
    clocks.start()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        y, _ = dec.decoder_iteration(x)
    ev1.record()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    clk = clocks.stop()
    launches = L.pgmoe_launch_count() + dec.replayed_kernels - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms], device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    # end to end: pinned host tokens in (into the iteration's input buffer),
    # result out, every step
    y_host = torch.empty_like(x_host).pin_memory()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x.copy_(x_host, non_blocking=True)
        y, _ = dec.decoder_iteration(x)
        y_host.copy_(y, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    t = torch.tensor([e2e_s], device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    e2e_s = float(t.item())
    nb = cfg.num_blocks
    # roofline of the dominant kernel (the expert FFN launch, up + down over
    # the rank's active local experts): one eager iteration with CUDA events
    # on the launching stream around each launch
    dec.use_graph, use_graph = False, dec.use_graph
    dec.ffn_events = []
    dec.decoder_iteration(x)
    torch.cuda.synchronize()
    evs, dec.ffn_events, dec.use_graph = dec.ffn_events, None, use_graph
    d, f = cfg.d_model, cfg.d_ff
    rows = world * T  # packed rows per launch (cap per peer)
    alg = [int(n.item()) * 2 * d * f * 2 + rows * (d * 2 + f * 2 * 2 + d * 4) for _, _, n in evs]
    us = [a.elapsed_time(b) * 1e3 for a, b, _ in evs]
    hbm_peak, _, peak_kind = peaks()
    achieved = sum(alg) / (sum(us) * 1e-6) / 1e9 if us and sum(us) > 0 else None
    out = {
        "metric": METRIC, "value": round(T * world / (ms * 1e-3), 3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference RNG weights/tokens, SURVEY §8(d))",
        "config": {"workload": f"Switch-{args.preset} expert-parallel x{world} (BASELINE configs[4])",
                   "preset": args.preset, "placement": "resident-sharded", "tokens_per_rank": T,
                   "global_batch": T * world, "num_blocks": nb, "parallelism": f"ep{world}",
                   "exchange": "NCCL all_to_all_single dispatch + combine per block",
                   "l2": "per-step expert bytes >> 126 MB L2", "kernel": args.kernel},
        "per_block_latency_ms": round(ms / nb, 4),
        "e2e": {"value": round(T * world / e2e_s, 3), "unit": "tokens/s",
                "h2d_bytes_per_step": T * cfg.d_model * 4, "d2h_bytes_per_step": T * cfg.d_model * 4},
        "gpu_launches": int(launches), "clocks": clk, "setup_s": round(setup_s, 2),
        "roofline": {"bound": "hbm", "kernel": "expert FFN launch (up + down, local experts), rank 0",
                     "achieved": round(achieved, 1) if achieved else None, "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4) if achieved else None, "traffic": None,
                     "peak_kind": peak_kind, "peak_note": PEAK_NOTE if peak_kind == "measured" else None,
                     "algorithmic_bytes_per_launch": int(sum(alg) / max(len(alg), 1)),
                     "avg_launch_us": round(sum(us) / max(len(us), 1), 2)},
    }
    dec.close()
    return out


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return None
    nth = os.cpu_count() or 1
    sample = args.cpu_sample or getattr(args, "tokens", 256)  # the whole batch: same config as our arm
    times = cpu_reference_run(args.preset, "bf16", sample, args.steps, min(args.warmup, 1), nth)
    s = statistics.mean(times)
    v = sample / s
    p = PRESETS[args.preset]
    return {
        "metric": METRIC, "impl": "reference", "value": round(v, 4), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(s * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference RNG weights rounded to bf16, SURVEY §8(d) tokens)",
        "config": {"workload": workload_name(args.preset, getattr(args, "placement", "offloaded"),
                                             getattr(args, "tokens", 256)),
                   "preset": args.preset, "tokens_per_step": sample, "num_blocks": p["num_blocks"],
                   "host": "reference CPU path on host cores, bounded sample per step"},
        "cpu_baseline": {"value": round(v, 4), "unit": "tokens/s", "cores": nth, "kind": "port",
                         "sample": f"{sample} tokens x 1 decoder iteration ({p['num_blocks']} blocks) per step; "
                                   f"oracle C restatement of moesim (bit-exact vs the reference on its golden "
                                   f"fixtures), {nth} threads"},
        "e2e": {"value": round(v, 4), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--preset", choices=sorted(PRESETS), default="large128")
    ap.add_argument("--placement", choices=["offloaded", "resident"], default="offloaded")
    ap.add_argument("--kernel", choices=["auto", "simt", "tcgen05"], default="auto")
    ap.add_argument("--dtype", choices=["bf16", "f32"], default="bf16",
                    help="weight dtype (f32: BASELINE configs[0]-style fp32 weights on the SIMT kernels)")
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity check after the timed region")
    ap.add_argument("--mode", choices=["auto", "single", "ep"], default="auto",
                    help="auto: offloaded single-GPU at N=1, expert-parallel at N>1")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # stdout carries exactly the one JSON line: anything native libraries
    # print there (NCCL's version banner) goes to stderr instead
    json_out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), file=json_out, flush=True)
        return
    mode = args.mode if args.mode != "auto" else ("ep" if world > 1 else "single")
    if world > 1 or mode == "ep":
        import torch
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        torch.distributed.init_process_group("nccl", rank=rank, world_size=world)
    out = run_ep(args, rank, world) if mode == "ep" else run_ours(args, rank, world)
    if rank == 0:
        print(json.dumps(out), file=json_out, flush=True)
    if world > 1 or mode == "ep":
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
