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

    def run(tag, arglist, layers, per_launch_events, sampler=False, pace=None):
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
                if pace == "event" and k >= 2:
                    evs[k - 2][1].synchronize()
                elif pace == "sleep":
                    time.sleep(0.0004)
                if per_launch_events:
                    evs[k][0].record()
                if pace == "python":
                    kp, vp = W.layer_pools(i, 0)
                    dec.decode(W.q_in[i], kp, vp, W.seq_lens, page_table=W.page_table,
                               max_len=W.max_len, out=W.out[i], ctx=W.ctx, split_tokens=W.chunk,
                               k_new=W.kn_in[i], v_new=W.vn_in[i])
                else:
                    _lib.check(lib.lam_decode(W.ctx.handle, arglist[i], sp))
                if per_launch_events:
                    evs[k][1].record()
                k += 1
        t1.record()
        torch.cuda.synchronize()
        if smp:
            print("   clocks", smp.stop())
        per = t0.elapsed_time(t1) / (len(layers) * a.reps)
        kern = (sum(e0.elapsed_time(e1) for e0, e1 in evs) / len(evs)) if per_launch_events else per
        gbs = W.decode_bytes_per_launch / (kern / 1e3) / 1e9
        print(f"{tag:38s} per-launch {per * 1e3:7.1f} us  kernel {kern * 1e3:7.1f} us  {gbs:6.0f} GB/s",
              flush=True)

    allL = list(range(L))
    for r in range(2):
        run(f"fast enqueue [{r}]", args, allL, True)
        run(f"paced: event 2 behind [{r}]", args, allL, True, pace="event")
        run(f"paced: sleep 0.4 ms [{r}]", args, allL, True, pace="sleep")
        run(f"paced: python make_args [{r}]", args, allL, True, pace="python")
        run(f"fast enqueue + sampler thread [{r}]", args, allL, True, sampler=True)

if __name__ == "__main__":
    main()
