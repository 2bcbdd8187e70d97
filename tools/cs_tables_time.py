import sys, time
sys.path.insert(0, ".")
import torch
import paper_2206_00975_b200 as nsk
A = torch.randn(1, 1 << 24, dtype=torch.float64, device="cuda").t()
for i in range(3):
    S = nsk.SketchOperator.draw("countsketch", 4096, 1 << 24, 7 + i)
    t = time.perf_counter()
    nsk.apply(S, A)
    torch.cuda.synchronize()
    print("first apply (tables) %.1f ms" % ((time.perf_counter() - t) * 1e3))
