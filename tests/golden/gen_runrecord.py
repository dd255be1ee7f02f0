"""Golden run record produced by the REFERENCE (mpsim.bench.fit): a small MLP
in f16 with initial scale 2^30 (so early steps overflow and are skipped) and
growth_interval 4 (so the scale also grows), with per-step parameter
checksums.  Writes tests/golden/runrecord_ref.csv (the reference's own CSV
writer) and runrecord_ref_params.npz (the final f32 model + its checksum), which
tests/test_runrecord_cpu.py replays and re-digests with
paper_2507_03312_b200.runrecord.

    python tests/golden/gen_runrecord.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from mpsim import bench  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    cfg = bench.RunConfig(precision="f16", steps=40, batch_size=16, seed=3, model="mlp", feature_dim=8,
                          num_classes=3, lr=1e-2, loss_scale_init=2.0 ** 30, growth_interval=4, debug_checksums=True)
    records, model = bench.fit(cfg)
    bench.write_csv(records, str(OUT / "runrecord_ref.csv"), debug_checksums=True)
    leaves = bench._all_tensor_leaves(model)
    np.savez_compressed(OUT / "runrecord_ref_params.npz", checksum=np.array(bench.param_checksum(model)),
                        paths=np.array([p for p, _ in leaves]),
                        dtypes=np.array([t.dtype.value for t, in [(l,) for _, l in leaves]]),
                        **{f"leaf{i}": np.asarray(t.payload, np.float32) for i, (_, t) in enumerate(leaves)})
    print("skipped", sum(1 for r in records if not r.grads_finite), "of", len(records),
          "scales", sorted(set(r.scale for r in records)))


if __name__ == "__main__":
    main()
