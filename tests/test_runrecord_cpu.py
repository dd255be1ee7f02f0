"""Run records against the reference's own output
(tests/golden/gen_runrecord.py runs mpsim.bench.fit): the CSV round-trips,
the replay accepts the reference's record (scale column = state machine on its
flags, skipped steps leave the checksum unchanged) and rejects tampered ones,
and param_checksum reproduces the reference's digest."""
from pathlib import Path

import numpy as np
import torch

from paper_2507_03312_b200 import runrecord as RR

GOLD = Path(__file__).resolve().parent / "golden"


def test_reference_record_replays():
    recs = RR.read_csv(str(GOLD / "runrecord_ref.csv"))
    assert len(recs) == 40 and sum(not r.grads_finite for r in recs) > 0
    rep = RR.replay(recs, init_scale=2.0 ** 30, growth_interval=4)
    assert rep.ok, rep
    assert rep.skipped == sum(not r.grads_finite for r in recs)


def test_replay_detects_tampering():
    recs = RR.read_csv(str(GOLD / "runrecord_ref.csv"))
    bad = [RR.StepRecord(**vars(r)) for r in recs]
    i = next(k for k, r in enumerate(bad) if r.grads_finite and k > 0)
    bad[i].scale *= 2.0
    assert i in RR.replay(bad, init_scale=2.0 ** 30, growth_interval=4).scale_mismatches
    bad = [RR.StepRecord(**vars(r)) for r in recs]
    j = next(k for k, r in enumerate(bad) if not r.grads_finite and k > 0)
    bad[j].param_checksum = "0" * 16
    assert j in RR.replay(bad, init_scale=2.0 ** 30, growth_interval=4).skip_changed_params


def test_csv_round_trip(tmp_path):
    recs = RR.read_csv(str(GOLD / "runrecord_ref.csv"))
    out = tmp_path / "r.csv"
    RR.write_csv(recs, str(out), debug_checksums=True)
    assert out.read_text() == (GOLD / "runrecord_ref.csv").read_text()


def test_param_checksum_matches_reference():
    z = np.load(GOLD / "runrecord_ref_params.npz")
    paths, dtypes = [str(p) for p in z["paths"]], [str(d) for d in z["dtypes"]]
    assert set(dtypes) == {"f32"}
    tree = {}
    for i, p in enumerate(paths):  # rebuild the nested dict the reference digested (dict order kept)
        node = tree
        parts = p.split(".")
        for k in parts[:-1]:
            node = node.setdefault(k, {})
        node[parts[-1]] = torch.from_numpy(z[f"leaf{i}"])
    assert RR.param_checksum(tree) == str(z["checksum"])
    # a half leaf digests as the reference's half tensor: dtype name + its f32 grid values
    import hashlib
    leaf = torch.from_numpy(z["leaf0"]).to(torch.bfloat16)
    h = hashlib.sha256()
    for part in (b"w", b"bf16", str(tuple(leaf.shape)).encode(), leaf.float().numpy().tobytes()):
        h.update(part)
    assert RR.param_checksum({"w": leaf}) == h.hexdigest()[:16]
