#!/usr/bin/env python
"""Benchmark of the B200-native MPX mixed-precision step.

Headline workload = BASELINE.json configs[1] ("fused mixed-precision step
microbench") with SURVEY.md §8(d)'s input recipe, used verbatim by BOTH arms:
the ViT-B/16 parameter pytree (152 leaves, 86,567,656 f32 params) drawn from
numpy default_rng(0) as N(0, 0.02^2), then the scaled gradients
N(0, (1e-3*2^15)^2) from the same generator rounded to the half format, m = v
= 0, loss scale 2^15, Adam lr 1e-3; +inf injected at steps = 3 (mod 10) into
blocks.5.fc1.w[17, 123] so every tenth step exercises skip + backoff.  One
step = K2 unscale+finite -> (N>1: finite-flag MIN all-reduce) -> K4 gated Adam
writing p32/m/v/p_half -> K3 adjust.  The f16 run is the headline, the bf16
run is the `bf16` sub-object (its own roofline).

Further sections (same JSON line): `vit_b16_train` (configs[2] at N=1: bf16
batch 256; configs[3] at N>1: f16 data parallel, per-GPU batch 256) and
`vit_l16_train` (configs[4]: f16 from a 2^32 loss scale, the device scale
trajectory replayed on the reference's state machine).

    python bench.py [--gpus N] [--steps K] [--warmup W]
    python bench.py --impl reference ...   # the reference (mpsim) on the host cores

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N ranks (one per GPU, NCCL); rank 0 prints
the one JSON line.  Units: GB/s of ALGORITHMIC traffic (30 B/param on a finite
step, 2 B/param on a skipped one).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ViT-B/16 mixed-precision train images/sec at 1/2/4/8 B200; fused MP-step GB/s vs HBM"
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
FALLBACK_BF16_TFLOPS = 1346.3
POISON_LEAF, POISON_INDEX = "blocks.5.fc1.w", (17, 123)
REF_DIR = ROOT / "baseline" / "_ref"
LR = 1e-3
INIT_SCALE = 2.0 ** 15
GRAD_STD = 1e-3 * 2 ** 15


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def tensor_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text()).get("bf16_tflops_sustained", FALLBACK_BF16_TFLOPS))
    return FALLBACK_BF16_TFLOPS


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def poisoned(i: int) -> bool:
    return i % 10 == 3


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.gpu = gpu_index
        self.path = ROOT / "gpurun_out" / f".clocks_{os.getpid()}_{id(self)}.csv"  # nested samplers

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001 - clocks are informative only
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return None
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6 and parts[0].isdigit():
                rows.append(parts)
        try:
            self.path.unlink()
        except OSError:
            pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in rows), "sm_max_mhz": int(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# the §8(d) input recipe (numpy; identical for both arms)
# ---------------------------------------------------------------------------
def recipe_host(shapes, rank: int = 0):
    """f32 params N(0, 0.02^2) and UNROUNDED scaled grads N(0, (1e-3*2^15)^2),
    from np.random.default_rng(0) in leaf order (params first).  Rank r > 0 of
    a data-parallel run draws its grads from default_rng((0, r))."""
    import numpy as np

    rng = np.random.default_rng(0)
    params = [rng.standard_normal(s, dtype=np.float32) * np.float32(0.02) for _, s in shapes]
    grng = rng if rank == 0 else np.random.default_rng((0, rank))
    grads = [grng.standard_normal(s, dtype=np.float32) * np.float32(GRAD_STD) for _, s in shapes]
    return params, grads


def poison_flat_index(shapes, leaf: str = POISON_LEAF):
    """(leaf index, flat index) of the injected +inf; a bounded sample without
    the leaf poisons its last leaf instead (flat index clipped)."""
    import math

    names = [n for n, _ in shapes]
    if leaf in names:
        i = names.index(leaf)
        cols = shapes[i][1][-1]
        return i, POISON_INDEX[0] * cols + POISON_INDEX[1]
    i = len(shapes) - 1
    return i, min(POISON_INDEX[0] * shapes[i][1][-1] + POISON_INDEX[1], math.prod(shapes[i][1]) - 1)


# ---------------------------------------------------------------------------
# the reference itself (mpsim, installed unmodified in baseline/_ref) on the host
# ---------------------------------------------------------------------------
def load_mpsim():
    if (REF_DIR / "mpsim" / "__init__.py").exists():
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        try:
            import mpsim  # noqa: F401

            return sys.modules["mpsim"]
        except Exception:  # noqa: BLE001 - fall back to the port
            return None
    return None


def _balanced_shards(sizes, n):
    order = sorted(range(len(sizes)), key=lambda i: -sizes[i])
    loads = [0] * n
    shards = [[] for _ in range(n)]
    for i in order:
        k = loads.index(min(loads))
        shards[k].append(i)
        loads[k] += sizes[i]
    return [sorted(s) for s in shards if s]


class MpsimStep:
    """The reference's own post-backward step — `LossScaling.unscale`,
    `all_finite`, `LossScaling.adjust`, `optimizer_update` (precision.py:145-173,
    tree.py:125-131, optim.py:100-113) and the `cast_tree(params, half)` that
    produces the next step's half working copy (precision.py:209) — over
    balanced leaf shards on a thread pool (numpy releases the GIL), the flags
    AND-ed across shards exactly as SURVEY.md §8(d) prescribes."""

    def __init__(self, mpsim, shapes, params, half: str, threads: int, lr: float = LR):
        self.M = mpsim
        self.half = mpsim.F16 if half == "f16" else mpsim.BF16
        self.paths = [n for n, _ in shapes]
        self.shards = _balanced_shards([p.size for p in params], max(1, threads))
        self.models = [{self.paths[i]: mpsim.tensor(params[i]) for i in sh} for sh in self.shards]
        self.states = [mpsim.adam_init(m, lr) for m in self.models]
        self.pool = ThreadPoolExecutor(max_workers=max(1, threads))
        self.threads = threads
        self.half_copy = None

    def grads(self, grads_f32):
        """Scaled grads as reference tensors of the half dtype (quantized by mpsim)."""
        return [{self.paths[i]: self.M.tensor(grads_f32[i], self.half) for i in sh} for sh in self.shards]

    def step(self, gshards, scaling):
        M = self.M

        def check(k):
            g32 = scaling.unscale(gshards[k])
            return g32, M.all_finite(g32)

        res = list(self.pool.map(check, range(len(self.shards))))
        fin = all(f for _, f in res)
        new_scaling = scaling.adjust(fin)

        def upd(k):
            self.models[k], self.states[k] = M.optimizer_update(self.models[k], self.states[k], res[k][0], fin)
            return M.cast_tree(self.models[k], self.half)

        self.half_copy = list(self.pool.map(upd, range(len(self.shards))))
        return new_scaling, fin

    def close(self):
        self.pool.shutdown()


class PortStep:
    """Fallback when mpsim is not installed: the oracle port (same op order)."""

    def __init__(self, shapes, params, half: str, threads: int, lr: float = LR):
        import numpy as np

        from oracle import mpx_oracle as O

        self.O, self.half = O, half
        self.runner = O.ThreadedStep(params, [np.zeros_like(p) for p in params], [np.zeros_like(p) for p in params],
                                     threads, lr=lr, half_fmt=half)
        self.t = 0
        self.threads = threads

    def grads(self, grads_f32):
        return [self.O.quantize(g, self.half) for g in grads_f32]

    def step(self, g, state):
        state, self.t, fin = self.runner.step(g, state, self.t)
        return state, fin

    def close(self):
        self.runner.close()


def host_runner(shapes, params, half, threads):
    """(runner, initial scaling, kind): mpsim itself when installed, else the port."""
    mpsim = load_mpsim()
    if mpsim is not None:
        return MpsimStep(mpsim, shapes, params, half, threads), mpsim.LossScaling(INIT_SCALE), "reference"
    return PortStep(shapes, params, half, threads), (INIT_SCALE, 2.0, 0.5, 2000, 0, 1.0), "port"


def poison_host(gshards_or_list, runner, shapes, leaf_idx, flat):
    """A copy of the host grads with +inf at (leaf_idx, flat)."""
    import numpy as np

    if isinstance(runner, MpsimStep):
        path = runner.paths[leaf_idx]
        out = []
        for sh in gshards_or_list:
            if path in sh:
                sh = dict(sh)
                arr = np.array(sh[path].payload)
                arr.reshape(-1)[flat] = np.inf
                sh[path] = runner.M.tensor(arr, runner.half)
            out.append(sh)
        return out
    out = list(gshards_or_list)
    arr = out[leaf_idx].copy()
    arr.reshape(-1)[flat] = np.inf
    out[leaf_idx] = arr
    return out


def cpu_baseline_sample(half: str, steps: int = 2):
    """The reference (mpsim) on the box's host cores over the FULL ViT-B
    pytree with the §8(d) recipe, threaded over balanced leaf shards."""
    from oracle.mpx_oracle import vit_b16_leaf_shapes

    shapes = vit_b16_leaf_shapes()
    params, grads = recipe_host(shapes)
    cores = os.cpu_count() or 1
    runner, scaling, kind = host_runner(shapes, params, half, cores)
    g = runner.grads(grads)
    del grads
    scaling, _ = runner.step(g, scaling)  # warm-up
    t0 = time.perf_counter()
    for _ in range(steps):
        scaling, fin = runner.step(g, scaling)
        assert fin
    dt = (time.perf_counter() - t0) / steps
    runner.close()
    n = sum(p.size for p in params)
    src = "mpsim (the reference, unmodified, baseline/_ref)" if kind == "reference" else "numpy oracle port"
    return {"value": round(n * 30 / dt / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": kind,
            "sample": f"full ViT-B pytree ({n} params, 152 leaves), {steps} finite {half} steps of {src}: unscale -> "
                      f"all_finite -> adjust -> optimizer_update -> cast_tree(half), threaded over {cores} balanced "
                      f"leaf shards; {dt * 1e3:.1f} ms/step"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def mp_section(args, half_name, dev, ws, rank, group, barrier, max_over_ranks, shapes, params_np, grads_np):
    """configs[1] for one half format: timed device step, K4 alone, e2e."""
    import torch

    from paper_2507_03312_b200 import DynamicLossScaling, as_dtype
    from paper_2507_03312_b200 import kernels as K
    from paper_2507_03312_b200.step import FusedMPStep

    half = as_dtype(half_name)
    params = {path: torch.from_numpy(p).to(dev) for (path, _), p in zip(shapes, params_np)}
    step = FusedMPStep(params, lr=LR, half_dtype=half, scaling=DynamicLossScaling(INIT_SCALE, device=dev),
                       process_group=group)
    del params
    n = step.n_params
    g32 = [torch.from_numpy(g).to(dev) for g in grads_np]
    K.cast_into(g32, step.grad.views)  # K1: the recipe's rounding of the scaled grads to the half grid
    del g32
    clean = step.grad.buf
    li, flat = poison_flat_index(shapes)
    pois = clean.clone()
    pois[step.offsets[li] + flat] = float("inf")
    ptr = lambda i: pois.data_ptr() if poisoned(i) else clean.data_ptr()  # noqa: E731
    skipped = lambda a, b: sum(1 for i in range(a, b) if poisoned(i))  # noqa: E731
    K_, W = args.steps, args.warmup
    stream = torch.cuda.current_stream(dev)
    for i in range(W):
        step.step(ptr(i))
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib = step._lib
    n0 = lib.mpx_launch_count()
    e0.record(stream)
    for i in range(W, W + K_):
        step.step(ptr(i))
    e1.record(stream)
    launches = lib.mpx_launch_count() - n0
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    n_skip = skipped(W, W + K_)
    algo_bytes = n * (30 * (K_ - n_skip) + 2 * n_skip)
    # the dominant kernel (K4) timed alone with events on its launch stream
    k4 = []
    base = W + K_
    for i in range(base, base + K_):
        p = ptr(i)
        step.k2(p)
        if not poisoned(i):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step.k4(p)
            b.record(stream)
            k4.append((a, b))
        else:
            step.k4(p)
        step.k3()
    torch.cuda.synchronize()
    k4_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in k4))
    # end to end with HOST gradient buffers: pinned H2D of every step's grads on
    # a copy stream (double-buffered against the compute stream), then a D2H
    # read of (flag, used scale)
    host_clean = torch.empty(clean.numel(), dtype=clean.dtype, pin_memory=True)
    host_clean.copy_(clean)
    host_pois = torch.empty_like(host_clean, pin_memory=True)
    host_pois.copy_(pois)
    land = [clean, pois]
    cs = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    out_flag = torch.empty(K_, dtype=torch.int32, pin_memory=True)
    out_scale = torch.empty(K_, dtype=torch.float64, pin_memory=True)
    torch.cuda.synchronize()
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    cs.wait_stream(stream)
    base = W + 2 * K_
    for j in range(K_):
        i = base + j
        b = j % 2
        with torch.cuda.stream(cs):
            if j >= 2:
                cs.wait_event(consumed[b])
            land[b].copy_(host_pois if poisoned(i) else host_clean, non_blocking=True)
            copied[b].record(cs)
        stream.wait_event(copied[b])
        step.step(land[b].data_ptr())
        consumed[b].record(stream)
        out_flag[j].copy_(step.flag, non_blocking=True)
        out_scale[j].copy_(step.used_scale, non_blocking=True)
    s1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(s0.elapsed_time(s1))
    e2e_skip = skipped(base, base + K_)
    assert int(out_flag.numpy().sum()) == K_ - e2e_skip, "e2e flags disagree with the injected schedule"
    hbm, peak_src = peaks()
    k4_bytes = n * FusedMPStep.K4_BYTES
    achieved = k4_bytes / (k4_ms * 1e-3) / 1e9
    grad_bytes = clean.numel() * clean.element_size()
    e2e_bytes = n * (30 * (K_ - e2e_skip) + 2 * e2e_skip)
    traffic, tsrc = None, None
    tf = ROOT / "profiles" / "k4_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(half_name)
        tsrc = f"from_profile: ncu --set full dram__bytes_read+write of K4 at this size ({tf.relative_to(ROOT)})"
    out = {
        "value": round(ws * algo_bytes / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "ms_per_step": round(ms / K_, 5),
        "half": half_name, "params": n, "skipped_steps": n_skip, "grad_arena_bytes": grad_bytes,
        "roofline": {"bound": "hbm", "kernel": "optimizer_kernel (K4)", "achieved": round(achieved, 1), "peak": hbm,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "algorithmic_bytes_per_launch": k4_bytes, "k4_ms": round(k4_ms, 5), "traffic": traffic,
                     "traffic_source": tsrc},
        "e2e": {"value": round(ws * e2e_bytes / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": grad_bytes, "d2h_bytes_per_step": 12, "ms_per_step": round(e2e_ms / K_, 5),
                "path": "pinned host grads -> copy stream H2D (double-buffered) -> K2/K4/K3 -> D2H flag+scale"},
        "gpu_launches": int(launches),
    }
    del step, clean, pois, host_clean, host_pois, land
    torch.cuda.empty_cache()
    return out


def vit_section(args, cfg, B, half_name, dev, ws, rank, group, barrier, max_over_ranks, steps, warmup,
                init_scale=INIT_SCALE, trajectory_steps=0):
    """ViT training step (configs[2]/[3]: ViT-B/16; configs[4]: ViT-L/16 from
    2^32): per-GPU batch B, dynamic loss scaling + Adam, data parallel over
    the group.  With trajectory_steps, the first steps run eagerly from
    init_scale with the (flag, scale) of each recorded and replayed on the
    reference's LossScaling.adjust."""
    import torch

    from paper_2507_03312_b200 import LossScaling, as_dtype
    from paper_2507_03312_b200 import _native
    from paper_2507_03312_b200.trainer import ViTTrainer

    half = as_dtype(half_name)
    tr = ViTTrainer(cfg, B, half=half, lr=LR, device=dev, group=group, world_size=ws, seed=0,
                    loss_scale=init_scale, zero=args.zero and group is not None)
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    images = torch.randn(B, cfg.img, cfg.img, cfg.chans, generator=g, device=dev)
    labels = torch.randint(0, cfg.classes, (B,), generator=g, device=dev).to(torch.int32)
    stream = torch.cuda.current_stream(dev)
    traj = None
    if trajectory_steps:
        flags, scales = [], []
        for _ in range(trajectory_steps):
            tr.step(images, labels)
            torch.cuda.synchronize()
            flags.append(int(tr.mp.flag.item()))
            scales.append(float(tr.mp.used_scale.item()))
        s = LossScaling(init_scale)
        replays = True
        for f, sc in zip(flags, scales):
            replays &= s.loss_scale == sc
            s = s.adjust(bool(f))
        replays &= s.loss_scale == tr.scaling.to_host().loss_scale
        traj = {"init_scale": init_scale, "flags": flags, "scales": scales, "replays_on_adjust": bool(replays),
                "note": "used scale and finite flag of each step read from the device; replayed on "
                        "LossScaling.adjust (the reference's state machine, precision.py:156-173)"}
    # one CUDA graph per step, at N > 1 too (the NCCL bucket all-reduces, flag MIN and ZeRO
    # collectives are captured with the kernels; every rank captures the same sequence).
    # --dp-eager (or --no-graph) launches eagerly; a capture that fails on ANY rank makes
    # every rank fall back to eager launches (agreed through a MIN all-reduce), so the
    # ranks' collective sequences stay matched
    use_graph = not args.no_graph and not (group is not None and args.dp_eager)
    exec_note = None
    lib = _native.load()
    n0 = lib.mpx_launch_count()
    tr.step(images, labels)  # one eager step: the library kernels a step launches (a graph replays them)
    per_step = lib.mpx_launch_count() - n0
    if use_graph:  # the whole step as one CUDA graph (warm-up steps run inside capture())
        ok = 1
        try:
            tr.capture(images, labels, warmup=warmup)
        except Exception as e:  # noqa: BLE001 - agreed fallback below
            if group is None:
                raise
            ok, exec_note = 0, f"eager (graph capture failed: {type(e).__name__})"
            print(f"bench.py: rank {rank}: data-parallel graph capture failed: {e!r}", file=sys.stderr, flush=True)
        if group is not None:
            import torch.distributed as dist
            t = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            if int(t.item()) == 0:
                use_graph, exec_note = False, exec_note or "eager (graph capture failed on another rank)"
    if use_graph:
        step = tr.replay
    else:
        for _ in range(warmup):
            tr.step(images, labels)
        step = lambda: tr.step(images, labels)  # noqa: E731
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clocks:  # this section's own clocks (power cap under GEMM load)
        e0.record(stream)
        for _ in range(steps):
            loss = step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    clk = clocks.summary()
    final_loss = float(loss.item())
    finite = bool(tr.grads_finite)
    # end to end: images + labels from pinned host memory every step (copy
    # stream, double-buffered), loss read back every step.  The images travel
    # in the half format the step computes in: the model's first op rounds
    # them to it anyway (cast_tree(args, half), precision.py:209-210), so half
    # host data is the same input bit for bit, at half the PCIe bytes
    from paper_2507_03312_b200 import kernels as K
    img_half = torch.empty(images.shape, dtype=half.torch, device=dev)
    K.cast_into([images], [img_half])  # K1, RNE: the rounding the trainer's own cast applies
    h_img = torch.empty(images.shape, dtype=half.torch, pin_memory=True)
    h_img.copy_(img_half)
    h_lab = torch.empty(labels.shape, dtype=torch.int32, pin_memory=True)
    h_lab.copy_(labels)
    d_img = [torch.empty_like(img_half), torch.empty_like(img_half)]
    d_lab = [torch.empty_like(labels), torch.empty_like(labels)]
    if use_graph:  # one captured step per input buffer (they share every state buffer)
        for b in range(2):
            d_img[b].copy_(img_half)
            d_lab[b].copy_(labels)
        gidx = [tr.capture(d_img[b], d_lab[b], warmup=1) for b in range(2)]
    out_loss = torch.empty(steps, dtype=torch.float32, pin_memory=True)
    cs = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    torch.cuda.synchronize()
    barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    cs.wait_stream(stream)
    for j in range(steps):
        b = j % 2
        with torch.cuda.stream(cs):
            if j >= 2:
                cs.wait_event(consumed[b])
            d_img[b].copy_(h_img, non_blocking=True)
            d_lab[b].copy_(h_lab, non_blocking=True)
            copied[b].record(cs)
        stream.wait_event(copied[b])
        l2 = tr.replay(gidx[b]) if use_graph else tr.step(d_img[b], d_lab[b])
        consumed[b].record(stream)
        out_loss[j].copy_(l2, non_blocking=True)
    s1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(s0.elapsed_time(s1))
    peak = tensor_peak()
    tflops = cfg.flops_per_image() * B / (ms / steps * 1e-3) / 1e12
    name = "ViT-L/16" if cfg.dim == 1024 else "ViT-B/16"
    out = {
        "metric": f"{name} mixed-precision train images/sec", "value": round(ws * B * steps / (ms * 1e-3), 1),
        "unit": "img/s", "ms_per_step": round(ms / steps, 3), "steps": steps, "warmup": warmup,
        "gpu_launches": int(per_step * steps), "kernels_per_step": int(per_step), "clocks": clk,
        "config": {"model": f"{name} 224x224 ({cfg.n_params() / 1e6:.1f}M params, cls token, 1000 classes)",
                   "per_gpu_batch": B, "global_batch": B * ws, "half": half_name,
                   "loss_scaling": f"dynamic, init 2^{int(round(__import__('math').log2(init_scale)))}",
                   "optimizer": "Adam lr 1e-3 (fused K4, f32 master)", "data": "synthetic N(0,1) images",
                   "parallelism": f"dp{ws}" + ((" ZeRO-1 (per-block NCCL reduce-scatter overlapped with backward, "
                                                "sharded K2/K4, half all-gather)" if args.zero else
                                                " (per-block NCCL grad all-reduce overlapped with backward)")
                                               if group is not None else ""),
                   "execution": "one CUDA graph per step" if use_graph else (exec_note or "eager stream-ordered launches"),
                   "l2": "activations >> 126 MB L2: no flush needed"},
        "roofline": {"bound": "tensor", "achieved": round(tflops, 1), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(tflops / peak, 4), "flops_per_image": cfg.flops_per_image(),
                     "note": "whole-step training FLOPs (3x forward GEMM+attention) / step time vs measured "
                             "sustained cuBLAS bf16"},
        "e2e": {"value": round(ws * B * steps / (e2e_ms * 1e-3), 1), "unit": "img/s",
                "h2d_bytes_per_step": h_img.numel() * h_img.element_size() + h_lab.numel() * 4,
                "d2h_bytes_per_step": 4, "inputs": f"{half_name} images (the step's first op rounds f32 to it) "
                                                  "+ i32 labels, pinned host memory"},
        "final_loss": round(final_loss, 5), "last_step_finite": finite, "loss_scale": tr.scaling.loss_scale,
    }
    if traj is not None:
        out["scale_trajectory"] = traj
    del tr, images, labels, d_img, d_lab, img_half
    torch.cuda.empty_cache()
    return out


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2507_03312_b200.vit_config import VIT_B16, VIT_L16

    ws, rank, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the GPU arm has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if ws > 1 or args.dp_path:
        if args.dp_path and ws == 1:  # validation: the data-parallel code path through NCCL, world size 1
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
        group = dist.group.WORLD

    def barrier():
        if group is not None:
            dist.barrier()

    def max_over_ranks(x):
        if group is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    shapes = VIT_B16.param_shapes()
    params_np, grads_np = recipe_host(shapes, rank)
    with ClockSampler(local) as clocks:
        mp = mp_section(args, args.half, dev, ws, rank, group, barrier, max_over_ranks, shapes, params_np, grads_np)
        other = "bf16" if args.half == "f16" else "f16"
        mp2 = None if args.no_second_half else mp_section(args, other, dev, ws, rank, group, barrier,
                                                          max_over_ranks, shapes, params_np, grads_np)
        del params_np, grads_np
        vit = vitl = None
        if not args.no_vit:
            # configs[2] is bf16 on one GPU, configs[3] fp16 data-parallel: auto picks by world size
            vit_half = args.vit_half or ("bf16" if group is None else "f16")
            vit = vit_section(args, VIT_B16, args.vit_batch, vit_half, dev, ws, rank, group, barrier,
                              max_over_ranks, args.vit_steps, args.vit_warmup)
        if not args.no_vit_l:
            vitl = vit_section(args, VIT_L16, args.vit_batch, "f16", dev, ws, rank, group, barrier, max_over_ranks,
                               args.vit_l_steps, args.vit_warmup, init_scale=2.0 ** 32,
                               trajectory_steps=args.vit_l_trajectory)
    clk = clocks.summary()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": mp["value"], "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mp["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "fused MP step (BASELINE configs[1], SURVEY §8d recipe): ViT-B/16 pytree, 152 leaves, "
                               f"{mp['params']} f32 params N(0,0.02^2) from numpy default_rng(0), {args.half} scaled "
                               "grads N(0,(1e-3*2^15)^2) from the same generator, m=v=0, scale 2^15, Adam lr 1e-3, "
                               "+inf injected at step%10==3 in blocks.5.fc1.w[17,123]; K2 unscale+finite -> K4 gated "
                               "Adam (p32,m,v,p_half) -> K3 adjust",
                   "params": mp["params"], "half": args.half, "grad_arena_bytes": mp["grad_arena_bytes"],
                   "l2": "working set 2.6 GB >> 126 MB L2: no flush needed",
                   "parallelism": f"dp{ws} replicas + finite-flag MIN all-reduce" if group is not None else "single GPU",
                   "skipped_steps": mp["skipped_steps"]},
        "roofline": mp["roofline"], "e2e": mp["e2e"], "gpu_launches": mp["gpu_launches"], "clocks": clk,
    }
    if mp2 is not None:
        line[mp2["half"]] = {k: mp2[k] for k in ("value", "unit", "ms_per_step", "skipped_steps", "roofline", "e2e",
                                                  "gpu_launches")}
    if vit is not None:
        line["vit_b16_train"] = vit
    if vitl is not None:
        line["vit_l16_train"] = vitl
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_sample(args.half)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# reference arm: the reference (mpsim) on the host cores
# ---------------------------------------------------------------------------
def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import math

    from oracle.mpx_oracle import vit_b16_leaf_shapes

    shapes_full = vit_b16_leaf_shapes()
    n_full = sum(math.prod(s) for _, s in shapes_full)
    # bounded sample per step: a prefix of the pytree sized so the whole
    # --steps/--warmup run stays within ~2 minutes (~50 Mparam/s threaded)
    budget = args.ref_sample_params or int(max(1e6, min(n_full, 100.0 * 50e6 / max(1, args.steps + args.warmup))))
    shapes, acc = [], 0
    for path, s in shapes_full:
        if acc >= budget:
            break
        shapes.append((path, s))
        acc += math.prod(s)
    params, grads = recipe_host(shapes)
    n = sum(p.size for p in params)
    cores = os.cpu_count() or 1
    runner, scaling, kind = host_runner(shapes, params, args.half, cores)
    clean = runner.grads(grads)
    del grads
    li, flat = poison_flat_index(shapes)
    pois = poison_host(clean, runner, shapes, li, flat)
    for i in range(args.warmup):
        scaling, _ = runner.step(pois if poisoned(i) else clean, scaling)
    t0 = time.perf_counter()
    n_skip = 0
    for i in range(args.warmup, args.warmup + args.steps):
        scaling, fin = runner.step(pois if poisoned(i) else clean, scaling)
        n_skip += 0 if fin else 1
    dt = time.perf_counter() - t0
    runner.close()
    value = n * (30 * (args.steps - n_skip) + 2 * n_skip) / dt / 1e9
    src = "mpsim, the reference package installed unmodified in baseline/_ref" if kind == "reference" else \
        "numpy oracle port (mpsim not installed)"
    sample = (f"{len(shapes)} leading leaves of the ViT-B pytree ({n} of {n_full} params) per step" if n < n_full
              else f"the full ViT-B pytree ({n} params, 152 leaves) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "fused MP step (BASELINE configs[1], SURVEY §8d recipe) on the host: unscale -> "
                               "all_finite -> adjust -> optimizer_update (Adam) -> cast_tree(half); same inputs, "
                               "poison schedule and loss-scale start as the GPU arm",
                   "params": n, "half": args.half, "parallelism": f"{cores} host threads over balanced leaf shards",
                   "source": src},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": kind,
                         "sample": f"{sample}, threaded over {cores} balanced leaf shards; {src}"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--half", choices=["f16", "bf16"], default="f16", help="headline MP-step half format")
    ap.add_argument("--no-second-half", action="store_true", help="skip the other half format's MP-step run")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-vit", action="store_true", help="skip the ViT-B/16 training section")
    ap.add_argument("--no-vit-l", action="store_true", help="skip the ViT-L/16 (configs[4]) section")
    ap.add_argument("--vit-batch", type=int, default=256)
    ap.add_argument("--vit-steps", type=int, default=10)
    ap.add_argument("--vit-l-steps", type=int, default=5)
    ap.add_argument("--vit-l-trajectory", type=int, default=16,
                    help="ViT-L eager steps from 2^32 whose (flag, scale) are recorded and replayed")
    ap.add_argument("--vit-warmup", type=int, default=3)
    ap.add_argument("--vit-half", choices=["f16", "bf16"], default=None,
                    help="ViT-B section half format (default: bf16 at 1 GPU = configs[2], f16 at N > 1 = configs[3])")
    ap.add_argument("--no-graph", action="store_true", help="ViT sections: eager launches instead of a CUDA graph")
    ap.add_argument("--zero", action="store_true", help="ViT sections at N > 1: ZeRO-1 sharded optimizer step")
    ap.add_argument("--dp-graph", action="store_true",
                    help="(default now) ViT sections at N > 1: the data-parallel step (NCCL collectives included) "
                         "captured as one CUDA graph")
    ap.add_argument("--dp-eager", action="store_true",
                    help="ViT sections at N > 1: eager stream-ordered launches instead of the captured graph")
    ap.add_argument("--dp-path", action="store_true",
                    help="validation: run the N > 1 code path (NCCL group, eager ViT steps, f16) at world size 1")
    ap.add_argument("--ref-sample-params", type=int, default=0,
                    help="reference arm: parameters per step sample (0 = auto-bounded)")
    ap.add_argument("--dry-run", action="store_true",
                    help="print each rank's (rank, world size, local rank) and exit (launcher check)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (rank 0 prints the line)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    ws, rank, local = dist_env()
    if ws != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch N ranks for --gpus N")
    if args.dry_run:
        print(json.dumps({"dry_run": True, "impl": args.impl, "rank": rank, "world_size": ws, "local_rank": local}),
              flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
