"""bench.py's JSON contract on the host: the reference arm (the reference's
algorithm on the host cores) prints one line with the contract's keys, and
the GPU arm refuses to run without a device (no CPU fallback)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup",
                          "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 1 and line["warmup"] == 3 and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_gpu_arm_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "no CUDA device" in (out.stdout + out.stderr)


def _lines(out):
    return [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]


def test_gpus_n_self_launches_n_ranks():
    """--gpus 2 without a torchrun environment re-launches bench.py under
    torch.distributed.run with two ranks (each binds its own LOCAL_RANK)."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _lines(out)
    assert sorted((d["rank"], d["local_rank"]) for d in lines) == [(0, 0), (1, 1)]
    assert all(d["world_size"] == 2 for d in lines)


def test_reference_arm_two_ranks_prints_once():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference", "--steps",
                          "2", "--warmup", "3", "--ref-sample-params", "1000000"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = _lines(out)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_world_size_must_match_gpus():
    import os
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_recipe_is_shared_by_both_arms():
    """Both arms draw the §8(d) inputs from the same function, over the same
    leaf list (the package's ViT-B tree == the oracle's)."""
    sys.path.insert(0, str(ROOT))
    import numpy as np

    import bench
    from oracle.mpx_oracle import vit_b16_leaf_shapes
    from paper_2507_03312_b200.vit_config import VIT_B16

    assert [(n, tuple(s)) for n, s in VIT_B16.param_shapes()] == [(n, tuple(s)) for n, s in vit_b16_leaf_shapes()]
    shapes = [("a", (3, 4)), ("blocks.5.fc1.w", (20, 200))]
    p1, g1 = bench.recipe_host(shapes)
    p2, g2 = bench.recipe_host(shapes)
    assert all(np.array_equal(a, b) for a, b in zip(p1 + g1, p2 + g2))
    assert bench.poison_flat_index(shapes) == (1, 17 * 200 + 123)
