import sys, time, torch
from pathlib import Path
sys.path.insert(0, str(Path.cwd()))
from paper_2507_03312_b200.trainer import ViTTrainer
from paper_2507_03312_b200.vit_config import VIT_B16
dev = torch.device("cuda", 0)
tr = ViTTrainer(VIT_B16, 256, half="f16", device=dev)
x = torch.randn(256, 224, 224, 3, device=dev); y = torch.randint(0, 1000, (256,), device=dev).to(torch.int32)
for _ in range(3): tr.step(x, y)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): tr.step(x, y)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0)/10:.2f} ms/step, wall {1e3*(t2-t0)/10:.2f} ms/step")
if "--profile" in sys.argv:
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5): tr.step(x, y)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)
