"""In-graph kernel timeline of the ViT-B/16 training step (CUPTI activity
records through torch.profiler: real concurrent timings, no serialization,
unlike ncu).  Prints busy time, the idle gaps between consecutive kernels and
the per-kernel-name totals of one replayed CUDA-graph step.

    python tools/timeline_vit.py [batch] [bf16|f16] [out.json]
"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import as_dtype  # noqa: E402
from paper_2507_03312_b200.trainer import ViTTrainer  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_B16  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    half = as_dtype(sys.argv[2] if len(sys.argv) > 2 else "bf16")
    out = sys.argv[3] if len(sys.argv) > 3 else None
    dev = torch.device("cuda", 0)
    tr = ViTTrainer(VIT_B16, B, half=half, device=dev)
    x = torch.randn(B, 224, 224, 3, device=dev)
    y = torch.randint(0, 1000, (B,), device=dev).to(torch.int32)
    tr.capture(x, y)
    for _ in range(5):
        tr.replay()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(10):
        tr.replay()
    ev1.record()
    torch.cuda.synchronize()
    step_ms = ev0.elapsed_time(ev1) / 10
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            tr.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    evs.sort(key=lambda e: e.time_range.start)
    # the last replay's kernels: split at the largest gaps (between replays)
    starts = [e.time_range.start for e in evs]
    n = len(evs) // 3
    step = evs[-n:]
    t0, t1 = step[0].time_range.start, max(e.time_range.end for e in step)
    busy, gaps, last_end = 0.0, [], t0
    per = defaultdict(lambda: [0, 0.0])
    for e in step:
        s, d = e.time_range.start, e.time_range.elapsed_us()
        if s > last_end:
            gaps.append((s - last_end, e.name))
        busy += max(0.0, e.time_range.end - max(s, last_end))
        last_end = max(last_end, e.time_range.end)
        per[e.name][0] += 1
        per[e.name][1] += d
    print(f"step (events, 10 replays) {step_ms:.3f} ms; profiled step span {(t1 - t0) / 1e3:.3f} ms, "
          f"{len(step)} kernels, busy {busy / 1e3:.3f} ms, idle {sum(g for g, _ in gaps) / 1e3:.3f} ms "
          f"in {len(gaps)} gaps")
    gaps.sort(reverse=True)
    print("largest gaps (us, before kernel):")
    for g, nm in gaps[:15]:
        print(f"  {g:7.2f}  {nm[:90]}")
    print("per kernel name (total us, count):")
    for nm, (c, d) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"  {d:9.1f}  {c:4d}  {nm[:100]}")
    if out:
        Path(out).write_text(json.dumps([{"name": e.name, "start": e.time_range.start - t0,
                                          "dur": e.time_range.elapsed_us()} for e in step]))


if __name__ == "__main__":
    main()
