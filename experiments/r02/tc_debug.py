import math, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2405_01814_b200 import decode as dec
from tests.helpers import make_dense, oracle_decode
B, Hkv, D, L = 1, 1, 128, 128
for G in (1, 8):
    q, k, v = make_dense(B, Hkv * G, Hkv, D, L, torch.bfloat16, seed=3)
    lens = torch.tensor([L], dtype=torch.int32, device="cuda")
    a = dec.decode(q, k, v, lens, kernel="gqa_tc", out_dtype=torch.float32)
    b = dec.decode(q, k, v, lens, kernel="gqa_mma", out_dtype=torch.float32)
    mean = v[0, 0].float().mean(0)
    torch.cuda.synchronize()
    print("G", G, "tc-mma", float((a - b).abs().max()), "tc-mean", float((a[0, 0] - mean).abs().max()),
          "mma-mean", float((b[0, 0] - mean).abs().max()))
    # weights: recover softmax weights by solving with V = identity-ish
    v2 = torch.zeros_like(v)
    for t in range(min(L, D)):
        v2[0, 0, t, t] = 1.0
    a2 = dec.decode(q, k, v2, lens, kernel="gqa_tc", out_dtype=torch.float32)
    b2 = dec.decode(q, k, v2, lens, kernel="gqa_mma", out_dtype=torch.float32)
    torch.cuda.synchronize()
    print(" tc weights[:8]", a2[0, 0, :8].tolist())
    print(" mma weights[:8]", b2[0, 0, :8].tolist())
    s = (q[0, 0].float() @ k[0, 0].float().T) / math.sqrt(D)
    print(" ref weights[:8]", torch.softmax(s, 0)[:8].tolist())
