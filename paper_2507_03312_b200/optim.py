"""Optimizers over parameter trees with a finite-gated update (mirror of
mpsim.optim), executed by K4 — one fused HBM pass per step.

    OptimizerState, adam_init, sgd_init   optim.py:20-55
    compute_updates                       optim.py:58-97
    optimizer_update                      optim.py:100-113

Numerics are the reference's to the bit: f32 moments, every operator one
correctly rounded f32 op in the reference's order, bias corrections
f32(1 - beta**t) from Python doubles with t counting applied steps only,
and p' = round_{p.dtype}(p + u) so half-precision master leaves stay half.

The step counter lives on the device ({step_count, scratch} int64[2]): a
skipped step (device flag == 0) leaves it, the moments and the parameters
bit-identical without the host ever looking at the flag.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import torch

from . import kernels as K
from .dtypes import is_float_leaf
from .precision import DeviceBool, ScaledGrads, _keep_type
from .tree import TreeError, float_leaves, tree_leaves, tree_map, tree_zip_map


@dataclass(frozen=True)
class OptimizerState:
    kind: str  # "sgd" | "adam"
    lr: float
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    counter: torch.Tensor | None = None  # device int64[2] {step_count, scratch}
    mu: object = None
    nu: object = None
    weight_decay: float = 0.0  # decoupled (AdamW); 0 = the reference's Adam

    @property
    def step_count(self) -> int:
        """Applied steps so far (reads the device counter: synchronises)."""
        return 0 if self.counter is None else int(self.counter[0].item())


def _device_of(params):
    for _, x in float_leaves(params):
        return x.device
    raise ValueError("params contain no float tensor leaves")


def _check_params(params):
    if not float_leaves(params):
        raise ValueError("params contain no float tensor leaves")


def _new_counter(device) -> torch.Tensor:
    return torch.zeros(2, dtype=torch.int64, device=device)


def _zero_moments(params):
    leaves = [x for _, x in float_leaves(params)]
    K.require_cuda(leaves, "adam_init")
    uniq = list({id(x): x for x in leaves}.values())
    bufs = K.arena_like(uniq, torch.float32)
    if bufs:
        bufs[0].untyped_storage().fill_(0)  # one memset for the whole arena
    m = {id(x): b for x, b in zip(uniq, bufs)}
    return tree_map(lambda x: m[id(x)] if is_float_leaf(x) else None, params)


def sgd_init(params, lr: float) -> OptimizerState:
    _check_params(params)
    return OptimizerState("sgd", lr, counter=_new_counter(_device_of(params)))


def adam_init(params, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
              weight_decay: float = 0.0) -> OptimizerState:
    _check_params(params)
    return OptimizerState("adam", lr, beta1, beta2, eps, counter=_new_counter(_device_of(params)),
                          mu=_zero_moments(params), nu=_zero_moments(params), weight_decay=weight_decay)


def adamw_init(params, lr: float, weight_decay: float = 0.01, beta1: float = 0.9, beta2: float = 0.999,
               eps: float = 1e-8) -> OptimizerState:
    """Adam with decoupled weight decay: p' = (p + u) + p*(-lr*wd).
    Extension beyond the reference (SPEC.md lists weight decay as a non-goal);
    weight_decay=0 is exactly adam_init."""
    return adam_init(params, lr, beta1, beta2, eps, weight_decay=weight_decay)


def _mode(state: OptimizerState) -> int:
    if state.kind == "adam":
        return 0
    if state.kind == "sgd":
        return 1
    raise ValueError(f"unknown optimizer kind {state.kind!r}")


def _hp(state):
    return K.adam_hparams(state.lr, state.beta1, state.beta2, state.eps, state.weight_decay)


def _bc(state, device):
    return K.bias_correction_table(state.beta1, state.beta2, device) if state.kind == "adam" else None


def _grad_source(grads):
    """(tree, host scale, device scale) — f32 grads need no unscale."""
    if isinstance(grads, ScaledGrads):
        return grads.tree, grads.scale, grads.d_scale
    return grads, 1.0, None


def _collect(state, grads_tree, model=None):
    """Aligned (param, grad, m, v) rows in traversal order for every float
    grad leaf, after the reference's structure checks (tree_zip_map raises
    TreeError with the diverging path, optim.py:80-81, 113)."""
    adam = state.kind == "adam"
    if adam:
        tree_zip_map(lambda a, b: None, state.mu, grads_tree)
        ms, vs = tree_leaves(state.mu), tree_leaves(state.nu)
    if model is not None:
        tree_zip_map(lambda a, b: None, model, grads_tree)
        ps = tree_leaves(model)
    rows = []
    for i, g in enumerate(tree_leaves(grads_tree)):
        if not is_float_leaf(g):
            continue
        p = ps[i] if model is not None else None
        if model is not None and not is_float_leaf(p):
            continue  # apply_leaf leaves non-tensor params alone (optim.py:108-109)
        m = ms[i] if adam else None
        v = vs[i] if adam else None
        if adam and not (is_float_leaf(m) and is_float_leaf(v)):
            raise TreeError("gradient leaf has no moment slot (params/grads structure mismatch)")
        rows.append((p, g, m, v))
    return rows


def compute_updates(state: OptimizerState, grads):
    """(updates, new state) without applying them (optim.py:58-97); the input
    state is left untouched (functional)."""
    mode = _mode(state)
    tree, scale, d_scale = _grad_source(grads)
    rows = _collect(state, tree)
    if not rows:
        return tree_map(lambda g: None, tree), replace(state, counter=state.counter.clone())
    dev = rows[0][1].device
    gs = [r[1] for r in rows]
    upd = K.arena_like(gs, torch.float32)
    counter = state.counter.clone()
    new_mu = new_nu = None
    if mode == 0:
        m2 = [r[2].clone() for r in rows]
        v2 = [r[3].clone() for r in rows]
    else:
        m2 = v2 = None
    K.optimizer_step(gs, gs, m2, v2, mode=mode, hp=_hp(state), counter=counter, bc_table=_bc(state, dev),
                     scale=scale, d_scale=d_scale, upd_out=upd)
    umap = {id(g): _keep_type(u, g) for g, u in zip(gs, upd)}
    updates = tree_map(lambda g: umap.get(id(g)) if is_float_leaf(g) else None, tree)
    if mode == 0:
        mmap = {id(r[2]): x for r, x in zip(rows, m2)}
        vmap = {id(r[3]): x for r, x in zip(rows, v2)}
        new_mu = tree_map(lambda x: mmap.get(id(x), x), state.mu)
        new_nu = tree_map(lambda x: vmap.get(id(x), x), state.nu)
    return updates, replace(state, counter=counter, mu=new_mu, nu=new_nu)


def optimizer_update(model, state: OptimizerState, grads, grads_finite, *, donate: bool = False,
                     half_copy=None):
    """One gated step (optim.py:100-113).

    grads_finite False (a host bool) returns (model, state) — the same
    objects, nothing launched.  A device flag (DeviceBool / int32 tensor)
    gates the fused K4 pass on the device instead.  By default the update is
    functional (fresh parameter and moment buffers, inputs untouched, like
    the reference); donate=True updates the buffers in place and returns
    the same objects.  `half_copy`, a tree of f16/bf16 tensors shaped like
    model, receives round_half(p') in the same pass (the working copy the
    next forward consumes)."""
    if isinstance(grads_finite, (bool,)) or (not isinstance(grads_finite, (DeviceBool, torch.Tensor))):
        if not bool(grads_finite):
            return model, state
        flag = None
    else:
        flag = grads_finite.tensor if isinstance(grads_finite, DeviceBool) else grads_finite
    mode = _mode(state)
    tree, scale, d_scale = _grad_source(grads)
    rows = _collect(state, tree, model)
    if not rows:
        return model, replace(state, counter=state.counter.clone()) if not donate else state
    dev = rows[0][0].device
    params = [r[0] for r in rows]
    gs = [r[1] for r in rows]
    halves = None
    if half_copy is not None:
        hrows = []
        tree_zip_map(lambda p, h: hrows.append((p, h)) if is_float_leaf(p) else None, model, half_copy)
        hmap = {id(p): h for p, h in hrows}
        halves = [hmap.get(id(p)) for p in params]
    if donate:
        new_p, m2, v2, counter = params, [r[2] for r in rows], [r[3] for r in rows], state.counter
        if mode == 1:
            m2 = v2 = None
    else:
        new_p = [p.clone() for p in params]
        m2 = [r[2].clone() for r in rows] if mode == 0 else None
        v2 = [r[3].clone() for r in rows] if mode == 0 else None
        counter = state.counter.clone()
    K.optimizer_step(new_p, gs, m2, v2, mode=mode, hp=_hp(state), counter=counter, bc_table=_bc(state, dev),
                     scale=scale, d_scale=d_scale, flag=flag, half_out=halves)
    if donate:
        return model, state
    pmap = {id(p): _keep_type(q, p) for p, q in zip(params, new_p)}
    new_model = tree_map(lambda x: pmap.get(id(x), x), model)
    new_mu = new_nu = None
    if mode == 0:
        mmap = {id(r[2]): x for r, x in zip(rows, m2)}
        vmap = {id(r[3]): x for r, x in zip(rows, v2)}
        new_mu = tree_map(lambda x: mmap.get(id(x), x), state.mu)
        new_nu = tree_map(lambda x: vmap.get(id(x), x), state.nu)
    return new_model, replace(state, counter=counter, mu=new_mu, nu=new_nu)
