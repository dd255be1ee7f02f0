"""Time the K5 tcgen05 GEMM on the ViT-B/16 (bs 256) linear shapes, fwd /
dgrad / wgrad, against torch.matmul (cuBLAS) on the same operands (the
forward as the engine runs it: on the K-major weight copy)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    dt = torch.bfloat16 if "--f16" not in sys.argv else torch.float16
    M = 256 * 197
    rows = []
    for name, K, N in [("qkv", 768, 2304), ("proj", 768, 768), ("fc1", 768, 3072), ("fc2", 3072, 768)]:
        x = torch.randn(M, K, device="cuda").to(dt)
        w = torch.randn(K, N, device="cuda").to(dt) * 0.03
        wt = w.t().contiguous()
        dy = torch.randn(M, N, device="cuda").to(dt)
        y = torch.empty(M, N, device="cuda", dtype=dt)
        dx = torch.empty(M, K, device="cuda", dtype=dt)
        dw = torch.empty(K, N, device="cuda", dtype=dt)
        fl = 2.0 * M * N * K
        for kind, ours, ref in [
            # the engine's forward reads K-major weight copies (linear_fwd_t)
            ("fwd", lambda: VK.linear_fwd_t(x, wt, out=y), lambda: torch.matmul(x, w, out=y)),
            ("dgrad", lambda: VK.linear_dgrad(dy, w, out=dx), lambda: torch.matmul(dy, w.t(), out=dx)),
            ("wgrad", lambda: VK.linear_wgrad(x, dy, out=dw), lambda: torch.matmul(x.t(), dy, out=dw)),
        ]:
            t1, t2 = timeit(ours), timeit(ref)
            rows.append({"gemm": f"{name}.{kind}", "M": M if kind != "wgrad" else K, "N": N if kind != "dgrad" else K,
                         "K": K if kind == "fwd" else (N if kind == "dgrad" else M),
                         "ours_ms": round(t1, 4), "ours_tflops": round(fl / t1 / 1e9, 1),
                         "cublas_ms": round(t2, 4), "cublas_tflops": round(fl / t2 / 1e9, 1)})
            print(json.dumps(rows[-1]), flush=True)
    tot1 = sum(r["ours_ms"] for r in rows)
    tot2 = sum(r["cublas_ms"] for r in rows)
    print(json.dumps({"per_layer_linear_ms_ours": round(tot1, 3), "per_layer_linear_ms_cublas": round(tot2, 3)}))


if __name__ == "__main__":
    main()
