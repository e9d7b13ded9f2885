import math, sys
import torch
sys.path.insert(0, ".")
from paper_2405_01814_b200 import decode as dec
B, Hkv, D, L = 1, 1, 128, 128
lens = torch.tensor([L], dtype=torch.int32, device="cuda")
v = torch.zeros((1, 1, L, D), device="cuda")
for t in range(L):
    v[0, 0, t, t] = 1.0
v = v.to(torch.bfloat16)
for j in (0, 8, 16, 32, 63, 64, 100, 127):
    q = torch.zeros((1, 1, D), device="cuda")
    q[0, 0, j] = 8.0
    k = torch.zeros((1, 1, L, D), device="cuda")
    for t in range(L):
        k[0, 0, t, j] = 1.0 if t % 2 else -1.0
    w = dec.decode(q.to(torch.bfloat16), k.to(torch.bfloat16), v, lens, kernel="gqa_tc", out_dtype=torch.float32)
    torch.cuda.synchronize()
    w = w[0, 0]
    print(f"dim {j}: odd/even weight ratio {float(w[1] / w[0]):.3f} (want {math.exp(16 / math.sqrt(128)):.3f}); "
          f"w[0:4] {[round(float(x), 5) for x in w[:4]]}", flush=True)
