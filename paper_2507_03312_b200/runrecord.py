"""Run records and replay.

The reference's training loop writes one CSV row per step —
``step,loss,scale,grads_finite,activation_bytes,wall_time_s[,param_checksum]``
(mpsim/bench.py:320-333, StepRecord bench.py:93-100) — with ``param_checksum``
a SHA-256 digest of every tensor leaf (bench.py:229-254).  This module writes
and reads the same format for GPU runs and replays a record:

* the scale column must follow the loss-scale state machine driven by the
  record's own ``grads_finite`` column (the reference's ``LossScaling.adjust``,
  precision.py:156-173, restated host-side in ``precision.LossScaling``), bit
  for bit — what tests/test_bench.py:84-95 does with ``simulate_scaling``;
* on a skipped step (``grads_finite`` false) the parameters must be unchanged:
  the checksum equals the previous step's (optim.py:102-103).

Checksums are computed exactly as the reference does for its immutable f32
payloads: a half leaf contributes the f32 values of its half grid, so a GPU
run's digest equals the reference's on the same values.
"""
from __future__ import annotations

import csv
import hashlib
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .precision import LossScaling

CSV_COLUMNS = ["step", "loss", "scale", "grads_finite", "activation_bytes", "wall_time_s"]

_DTYPE_NAME = {"torch.float16": "f16", "torch.bfloat16": "bf16", "torch.float32": "f32", "torch.int32": "i32"}


@dataclass
class StepRecord:
    step: int
    loss: float
    scale: float
    grads_finite: bool
    activation_bytes: int
    wall_time_s: float
    param_checksum: str | None = None


def _leaves(tree, path=()):
    if isinstance(tree, dict):
        for k, v in tree.items():
            yield from _leaves(v, path + (k,))
    elif isinstance(tree, (list, tuple)):
        for i, v in enumerate(tree):
            yield from _leaves(v, path + (i,))
    elif tree is not None and hasattr(tree, "shape") and hasattr(tree, "dtype"):
        yield ".".join(str(p) for p in path), tree


def _payload(leaf) -> tuple[str, tuple, bytes]:
    """(dtype name, shape, bytes of the reference's payload) of one leaf."""
    dt = str(leaf.dtype)
    if dt.startswith("torch."):
        name = _DTYPE_NAME[dt]
        host = leaf.detach()
        host = (host.float() if name != "i32" else host).cpu().numpy()
    else:  # numpy: f32 payload on the leaf's grid (f32 here)
        host = np.asarray(leaf)
        name = "i32" if host.dtype == np.int32 else "f32"
    arr = np.ascontiguousarray(host.astype(np.int32 if name == "i32" else np.float32, copy=False))
    return name, tuple(arr.shape), arr.tobytes()


def param_checksum(tree) -> str:
    """The reference's digest (bench.py:229-237) of every tensor leaf of `tree`:
    sha256 over path, dtype name, shape and the f32 (or i32) payload bytes."""
    h = hashlib.sha256()
    for path, leaf in _leaves(tree):
        name, shape, data = _payload(leaf)
        h.update(path.encode())
        h.update(name.encode())
        h.update(str(shape).encode())
        h.update(data)
    return h.hexdigest()[:16]


def write_csv(records: Iterable[StepRecord], path: str, debug_checksums: bool = False) -> None:
    """Same columns and number formatting as the reference (bench.py:323-333)."""
    columns = CSV_COLUMNS + (["param_checksum"] if debug_checksums else [])
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(columns)
        for r in records:
            row = [r.step, repr(float(r.loss)), repr(float(r.scale)), int(bool(r.grads_finite)),
                   int(r.activation_bytes), repr(float(r.wall_time_s))]
            if debug_checksums:
                row.append(r.param_checksum)
            w.writerow(row)


def read_csv(path: str) -> list[StepRecord]:
    out = []
    with open(path, encoding="utf-8", newline="") as fh:
        for row in csv.DictReader(fh):
            out.append(StepRecord(int(row["step"]), float(row["loss"]), float(row["scale"]),
                                  bool(int(row["grads_finite"])), int(row["activation_bytes"]),
                                  float(row["wall_time_s"]), row.get("param_checksum") or None))
    return out


@dataclass
class ReplayReport:
    steps: int
    skipped: int
    scale_mismatches: list[int]
    skip_changed_params: list[int]

    @property
    def ok(self) -> bool:
        return not self.scale_mismatches and not self.skip_changed_params


def replay(records: list[StepRecord], init_scale: float | None = None, growth_factor: float = 2.0,
           backoff_factor: float = 0.5, growth_interval: int = 2000, min_scale: float = 1.0,
           init_checksum: str | None = None) -> ReplayReport:
    """Check a run record: (1) every row's scale is the state machine's value
    before that step, driven by the record's own flags; (2) a skipped step
    leaves the parameter checksum unchanged (needs checksums; `init_checksum`
    is the digest before step 0)."""
    if not records:
        return ReplayReport(0, 0, [], [])
    s = LossScaling(records[0].scale if init_scale is None else init_scale, growth_factor, backoff_factor,
                    growth_interval, 0, min_scale)
    bad_scale, bad_skip = [], []
    prev = init_checksum
    for r in records:
        if r.scale != s.loss_scale:
            bad_scale.append(r.step)
        if not r.grads_finite and r.param_checksum is not None and prev is not None and r.param_checksum != prev:
            bad_skip.append(r.step)
        prev = r.param_checksum
        s = s.adjust(r.grads_finite)
    return ReplayReport(len(records), sum(1 for r in records if not r.grads_finite), bad_scale, bad_skip)
