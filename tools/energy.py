"""Energy per ViT-B/16 training step and per kernel class (NVML total-energy
counter), for the power-capped regime the step runs in (sw_power_cap, SM
clock ~1.55-1.7 GHz of 1.965 under GEMM load): there, step time ~ energy /
power cap, so a change that only hides latency (same work, same joules)
does not speed the step up — a change that removes work or bytes does.

    python tools/energy.py [step|kernels|all|cublas|attn] [bf16|f16] [seconds_per_item]

`step`: replays the captured step graph for ~N s; prints ms/step, J/step,
mean W, median SM MHz.  `kernels`: each kernel class of the step at the
ViT-B bs-256 shape, launched back to back for ~N s with the buffers of a real
step: us/launch, mJ/launch, W, MHz, and x launches/step -> J/step share.
One JSON line per item.
"""
import json
import statistics
import sys
import threading
import time
from pathlib import Path

import pynvml
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_03312_b200 import as_dtype  # noqa: E402
from paper_2507_03312_b200 import kernels as K_  # noqa: E402
from paper_2507_03312_b200 import vit_kernels as VK  # noqa: E402
from paper_2507_03312_b200.trainer import ViTTrainer  # noqa: E402
from paper_2507_03312_b200.vit_config import VIT_B16  # noqa: E402


class Meter:
    def __init__(self, idx=0):
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
        self.samples = []
        self._stop = threading.Event()

    def _poll(self):
        while not self._stop.is_set():
            self.samples.append((pynvml.nvmlDeviceGetPowerUsage(self.h) / 1e3,
                                 pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)))
            time.sleep(0.02)

    def run(self, fn, seconds):
        """fn() enqueues one unit; returns (units, ms/unit, J/unit, W, MHz)."""
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        # calibrate the units per ~seconds
        t = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        per = e0.elapsed_time(e1) / 5
        n = max(10, int(seconds * 1e3 / max(per, 1e-3)))
        self.samples, self._stop = [], threading.Event()
        th = threading.Thread(target=self._poll, daemon=True)
        j0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(self.h)  # mJ
        th.start()
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        j1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(self.h)
        self._stop.set()
        th.join()
        ms = e0.elapsed_time(e1)
        loaded = self.samples[len(self.samples) // 5:] or self.samples
        return (n, ms / n, (j1 - j0) / 1e3 / n, statistics.mean(p for p, _ in loaded),
                statistics.median(c for _, c in loaded))


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    half = as_dtype(sys.argv[2] if len(sys.argv) > 2 else "bf16")
    secs = float(sys.argv[3]) if len(sys.argv) > 3 else 4.0
    dev = torch.device("cuda", 0)
    B = 256
    tr = ViTTrainer(VIT_B16, B, half=half, device=dev)
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(B, 224, 224, 3, device=dev, generator=g)
    y = torch.randint(0, 1000, (B,), device=dev, generator=g).to(torch.int32)
    tr.capture(x, y)
    m = Meter(0)

    def emit(name, per_step, res):
        n, ms, j, w, mhz = res
        print(json.dumps({"item": name, "launches_per_step": per_step, "us": round(ms * 1e3, 2),
                          "mJ": round(j * 1e3, 3), "W": round(w, 1), "sm_mhz": mhz,
                          "J_per_step": round(j * per_step, 4), "ms_per_step": round(ms * per_step, 3),
                          "units_timed": n}), flush=True)

    if mode == "cublas":  # plain GEMMs of the step's shapes: ours vs cuBLAS (torch.matmul), same layouts
        M = 50432
        for name, K, N_ in (("qkv fwd", 768, 2304), ("proj fwd", 768, 768), ("fc1 fwd", 768, 3072),
                            ("fc2 fwd", 3072, 768)):
            a = torch.randn(M, K, device=dev).to(half.torch)
            wt = (torch.randn(N_, K, device=dev) / K ** 0.5).to(half.torch)
            c = torch.empty(M, N_, device=dev, dtype=half.torch)
            fl = 2.0 * M * K * N_
            for impl, fn in (("mpx", lambda: VK.linear_fwd_t(a, wt, out=c)),
                             ("cublas", lambda: torch.matmul(a, wt.t(), out=c))):
                n, ms, j, w, mhz = m.run(fn, secs)
                print(json.dumps({"item": f"{name} [{M}x{K}]x[{K}x{N_}] {impl}", "us": round(ms * 1e3, 2),
                                  "mJ": round(j * 1e3, 3), "W": round(w, 1), "sm_mhz": mhz,
                                  "GFLOP_per_J": round(fl / 1e9 / j, 1), "TFLOPs": round(fl / ms / 1e9, 1)}),
                      flush=True)
        return
    if mode == "attn":  # fused attention fwd+bwd vs cuDNN SDPA fwd+bwd, same shape, steady state
        import torch.nn.functional as F
        from torch.nn.attention import SDPBackend, sdpa_kernel
        S_, H_, hd_ = 197, 12, 64
        D_ = H_ * hd_
        qkv = torch.randn(B * S_, 3 * D_, device=dev).to(half.torch)
        dO = torch.randn(B * S_, D_, device=dev).to(half.torch)
        O_ = torch.empty(B * S_, D_, device=dev, dtype=half.torch)
        dqkv = torch.empty_like(qkv)
        ps = torch.empty(VK.attention_psave_bytes(B, S_, H_), dtype=torch.uint8, device=dev)
        sc = hd_ ** -0.5

        def ours():
            VK.attention_fwd(qkv, B, S_, H_, hd_, sc, out=O_, p_save=ps)
            VK.attention_bwd(qkv, dO, B, S_, H_, hd_, sc, dqkv=dqkv, p_saved=ps)
        q, k, v = (t.detach().requires_grad_() for t in qkv.view(B, S_, 3, H_, hd_).permute(2, 0, 3, 1, 4).unbind(0))
        dOv = dO.view(B, S_, H_, hd_).transpose(1, 2)

        def cudnn():
            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                out = F.scaled_dot_product_attention(q, k, v, scale=sc)
                torch.autograd.grad(out, (q, k, v), dOv)
        def ours_f():
            VK.attention_fwd(qkv, B, S_, H_, hd_, sc, out=O_, p_save=ps)

        def ours_b():
            VK.attention_bwd(qkv, dO, B, S_, H_, hd_, sc, dqkv=dqkv, p_saved=ps)
        cs_out = torch.empty(3 * D_, dtype=half.torch, device=dev)
        cs_ws = torch.empty(B * 3 * D_, dtype=torch.float32, device=dev)
        cs_ws2 = torch.empty(1 << 22, dtype=torch.float32, device=dev)

        def ours_b_cs():  # with the in-kernel qkv-bias gradient (column sums of dqkv), as the engine runs it
            VK.attention_bwd(qkv, dO, B, S_, H_, hd_, sc, dqkv=dqkv, p_saved=ps, colsum_out=cs_out, colsum_ws=cs_ws)

        def ours_b_sep():  # the same bias gradient by a separate column-sum pass over dqkv
            from paper_2507_03312_b200 import _native as NN
            VK.attention_bwd(qkv, dO, B, S_, H_, hd_, sc, dqkv=dqkv, p_saved=ps)
            NN.check(NN.load().mpx_colsum(VK._CODE[half.torch], dqkv.data_ptr(), 3 * D_, 0, B * S_, 3 * D_, 1,
                                          cs_ws2.data_ptr(), cs_ws2.numel(), cs_out.data_ptr(), 3 * D_,
                                          VK._CODE[half.torch], 1.0, K_.stream_handle(dev)), "colsum")
        items = (("mpx fused attention fwd+bwd", ours), ("cuDNN SDPA fwd+bwd", cudnn))
        if len(sys.argv) > 4 and sys.argv[4] == "split":
            items = (("mpx fused attention fwd", ours_f), ("mpx fused attention bwd", ours_b))
        if len(sys.argv) > 4 and sys.argv[4] == "colsum":
            items = (("bwd, no bias grad", ours_b), ("bwd + in-kernel bias grad", ours_b_cs),
                     ("bwd + separate colsum pass", ours_b_sep))
        for name, fn in items:
            n, ms, j, w, mhz = m.run(fn, secs)
            print(json.dumps({"item": name, "us": round(ms * 1e3, 2), "mJ": round(j * 1e3, 3), "W": round(w, 1),
                              "sm_mhz": mhz}), flush=True)
        return
    if mode in ("step", "all"):
        emit("step (CUDA graph replay)", 1, m.run(tr.replay, secs * 2))
    if mode not in ("kernels", "all"):
        return
    e = tr.engine
    P, G = tr.P, tr.G
    D, M, H, S, hd = e.D, e.M, e.H, e.S, e.hd
    q = "blocks.0."
    wt = e._wt[0]
    scale = hd ** -0.5
    items = [
        ("ln_fwd (standalone: block 0's LN1, ln_f)", 2 if e.ln_fold else 25,
         lambda: e._ln_fwd(e.x[0], D, P[q + "ln1.g"], P[q + "ln1.b"], e.a[0], D, e.mu1[0], e.rs1[0], M)),
        ("qkv fwd GEMM (+bias)", 12, lambda: VK.linear_fwd_t(e.a[0], wt["qkv"], bias=P[q + "qkv.b"], out=e.qkv[0])),
        ("attention fwd (P saved)", 12, lambda: VK.attention_fwd(e.qkv[0], B, S, H, hd, scale, out=e.O[0],
                                                                  p_save=e.attn_p[0])),
        ("proj fwd GEMM (+bias+res" + (", +LN2 fused)" if e.ln_fold else ")"), 12,
         lambda: VK.linear_fwd_t(e.O[0], wt["proj"], bias=P[q + "proj.b"], residual=e.x[0], out=e.xm[0],
                                 ln=(P[q + "ln2.g"], P[q + "ln2.b"], e.bn[0], e.mu2[0], e.rs2[0], 1e-5)
                                 if e.ln_fold else None)),
        ("fc1 fwd GEMM (+bias, GELU, aux out)", 12,
         lambda: VK.linear_fwd_t(e.bn[0], wt["fc1"], bias=P[q + "fc1.b"], act=VK.ACT_GELU_D, aux=e.pre[0], out=e.h[0])),
        ("fc2 fwd GEMM (+bias+res" + (", +next LN1 fused)" if e.ln_fold else ")"), 12,
         lambda: VK.linear_fwd_t(e.h[0], wt["fc2"], bias=P[q + "fc2.b"], residual=e.xm[0], out=e.x[1],
                                 ln=(P["blocks.1.ln1.g"], P["blocks.1.ln1.b"], e.a[1], e.mu1[1], e.rs1[1], 1e-5)
                                 if e.ln_fold else None)),
        ("fc2 wgrad GEMM", 12, lambda: VK.linear_wgrad(e.h[0], e.dX, out=G[q + "fc2.w"])),
        ("fc2 dgrad GEMM (GELU' aux in, colsum)", 12,
         lambda: VK.linear_dgrad(e.dX, P[q + "fc2.w"], aux=e.pre[0], out=e.dpre, colsum_out=G[q + "fc1.b"],
                                 colsum_ws=e.ws, aux_act=VK.ACT_MUL_AUX)),
        ("fc1 wgrad GEMM", 12, lambda: VK.linear_wgrad(e.bn[0], e.dpre, out=G[q + "fc1.w"])),
        ("fc1 dgrad GEMM", 12, lambda: VK.linear_dgrad(e.dpre, P[q + "fc1.w"], out=e.dA)),
        ("ln_bwd2", 25, lambda: e._ln_bwd2(e.xm[0], D, P[q + "ln2.g"], e.mu2[0], e.rs2[0], e.dA, D, e.dX, e.dXm, D,
                                          G[q + "ln2.g"], G[q + "ln2.b"], G[q + "proj.b"], M)),
        ("proj wgrad GEMM", 12, lambda: VK.linear_wgrad(e.O[0], e.dXm, out=G[q + "proj.w"])),
        ("proj dgrad GEMM", 12, lambda: VK.linear_dgrad(e.dXm, P[q + "proj.w"], out=e.dO)),
        ("attention bwd (P reloaded)", 12, lambda: VK.attention_bwd(e.qkv[0], e.dO, B, S, H, hd, scale,
                                                                     dqkv=e.dqkv, p_saved=e.attn_p[0],
                                                                     colsum_out=G[q + "qkv.b"], colsum_ws=e.ws)),
        ("qkv wgrad GEMM", 12, lambda: VK.linear_wgrad(e.a[0], e.dqkv, out=G[q + "qkv.w"])),
        ("qkv dgrad GEMM", 12, lambda: VK.linear_dgrad(e.dqkv, P[q + "qkv.w"], out=e.dA)),
        ("MP step (K2+K4+K3)", 1, lambda: tr.mp.step()),
    ]
    for name, n, fn in items:
        emit(name, n, m.run(fn, secs))


if __name__ == "__main__":
    main()
