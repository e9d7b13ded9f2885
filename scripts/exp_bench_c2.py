"""Diagnose the gap between bench.py's C2 decode launches and exp_decode's: the bench Workload's
own launches timed several ways on one box.

    python scripts/exp_bench_c2.py [--workload c2]
"""
import argparse
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2405_01814_b200 import _lib, decode as dec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    device = torch.device("cuda", 0)
    torch.cuda.set_device(device)
    W = bench.Workload(bench.WORKLOADS[a.workload], 0, 1, device)
    lib, sp = _lib.load(), torch.cuda.current_stream().cuda_stream
    L = W.layers
    args = []
    for layer in range(L):
        kp, vp = W.layer_pools(layer, 0)
        x, _ = dec.make_args(W.q_in[layer], kp, vp, W.seq_lens, page_table=W.page_table,
                             max_len=W.max_len, out=W.out[layer], split_tokens=W.chunk,
                             k_new=W.kn_in[layer], v_new=W.vn_in[layer])
        args.append(x)
    args_nf = []
    for layer in range(L):
        kp, vp = W.layer_pools(layer, 0)
        x, _ = dec.make_args(W.q_in[layer], kp, vp, W.seq_lens, page_table=W.page_table,
                             max_len=W.max_len, out=W.out[layer], split_tokens=W.chunk)
        args_nf.append(x)

    def run(tag, arglist, layers, per_launch_events, sampler=False):
        for _ in range(2):
            for i in layers:
                _lib.check(lib.lam_decode(W.ctx.handle, arglist[i], sp))
        torch.cuda.synchronize()
        smp = None
        if sampler:
            smp = bench.ClockSampler(0)
            smp.start()
            time.sleep(0.3)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(len(layers) * a.reps)]
        k = 0
        t0.record()
        for _ in range(a.reps):
            for i in layers:
                if per_launch_events:
                    evs[k][0].record()
                _lib.check(lib.lam_decode(W.ctx.handle, arglist[i], sp))
                if per_launch_events:
                    evs[k][1].record()
                k += 1
        t1.record()
        torch.cuda.synchronize()
        if smp:
            smp.stop()
        per = t0.elapsed_time(t1) / (len(layers) * a.reps)
        kern = (sum(e0.elapsed_time(e1) for e0, e1 in evs) / len(evs)) if per_launch_events else per
        gbs = W.decode_bytes_per_launch / (kern / 1e3) / 1e9
        print(f"{tag:38s} per-launch {per * 1e3:7.1f} us  kernel {kern * 1e3:7.1f} us  {gbs:6.0f} GB/s",
              flush=True)

    allL = list(range(L))
    run("fused, all layers, events", args, allL, True)
    run("fused, all layers, no events", args, allL, False)
    run("fused, all layers, events, sampler", args, allL, True, sampler=True)
    run("plain, all layers, events", args_nf, allL, True)
    run("fused, layers 0-1 only, events", args, [0, 1], True)
    run("plain, layers 0-1 only, events", args_nf, [0, 1], True)
    run("plain, layer 0 only, events", args_nf, [0], True)


if __name__ == "__main__":
    main()
