#!/bin/bash
# Diagnostic for the C3 N=4 host-buffer gap: box topology (NUMA affinity of each GPU) and host
# memory bandwidth; no code change.
mkdir -p gpurun_out
exec > gpurun_out/call69.log 2>&1
nvidia-smi topo -m
lscpu | grep -i "numa\|model name\|socket\|^cpu(s)"
python - <<'PY'
import torch, time
# pinned host -> device copy rate, one GPU alone, then all four at once (threads)
import threading
n = 256 << 20
def run(dev, res):
    torch.cuda.set_device(dev)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True); d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3): d.copy_(h, non_blocking=True)
        s.synchronize(); t = time.perf_counter()
        for _ in range(20): d.copy_(h, non_blocking=True)
        s.synchronize(); res[dev] = 20 * n / (time.perf_counter() - t) / 1e9
for devs in ([0], [0, 1], [0, 1, 2, 3]):
    res = {}
    ts = [threading.Thread(target=run, args=(i, res)) for i in devs]
    [t.start() for t in ts]; [t.join() for t in ts]
    print("h2d GB/s per GPU, concurrent", devs, {k: round(v, 1) for k, v in res.items()})
PY
