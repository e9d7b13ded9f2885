"""Stream memory-operation latency on B200 (diagnostic for the peer engine's model-worker relay).

Times chains of cuStreamWriteValue32 / cuStreamWaitValue32 on one GPU and across two GPUs
(flags in the peer's memory), with and without the write's system-scope memory barrier.
Run: [LAM_SIGNAL_NO_BARRIER=1] python experiments/r02/memop_latency.py   (1 or 2 visible GPUs)
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
from paper_2405_01814_b200 import _lib  # noqa: E402

ITERS = 400
LIB = _lib.load()
CTX = {}


def ctx(dev):
    if dev not in CTX:
        CTX[dev] = _lib.Context(dev)
    return CTX[dev]


def write(s, p, v, fl=None):
    arr = (C.c_void_p * 1)(p)
    _lib.check(LIB.lam_stream_signal(ctx(s.device.index).handle, arr, 1, v, s.cuda_stream))


def wait(s, p, v):
    arr = (C.c_void_p * 1)(p)
    _lib.check(LIB.lam_stream_wait(ctx(s.device.index).handle, arr, 1, v, s.cuda_stream))


def ptr(t, i=0):
    return t.data_ptr() + 4 * i


def timed(dev, streams, body):
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s in streams[1:]:
        s.wait_event(e0)
    body()
    for s in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(s)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) * 1000.0 / ITERS  # us per iteration


def main():
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    a, b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}
    tag = "nobarrier" if os.environ.get("LAM_SIGNAL_NO_BARRIER") == "1" else "default"
    for name, fl in ((tag, None),):
        f = torch.zeros(8, dtype=torch.int32, device=dev)
        res[f"write_chain_{name}"] = timed(dev, [a], lambda: [write(a, ptr(f), i + 1, fl) for i in range(ITERS)])
        f.zero_()

        def selfwait():
            for i in range(ITERS):
                write(a, ptr(f), i + 1, fl)
                wait(a, ptr(f), i + 1)
        res[f"write_wait_same_stream_{name}"] = timed(dev, [a], selfwait)
        f.zero_()

        def pingpong(fa, fb):
            for i in range(ITERS):
                write(a, fa, i + 1, fl)     # A -> B
                wait(b, fa, i + 1)
                write(b, fb, i + 1, fl)     # B -> A
                wait(a, fb, i + 1)
        res[f"pingpong_2streams_{name}"] = timed(dev, [a, b], lambda: pingpong(ptr(f, 0), ptr(f, 4)))
        f.zero_()

        x = torch.zeros(1, device=dev)

        def kernel_then_signal():
            with torch.cuda.stream(a):
                for i in range(ITERS):
                    x.add_(1.0)
                    write(a, ptr(f), i + 1, fl)
        res[f"kernel_then_write_{name}"] = timed(dev, [a], kernel_then_signal)

        def kernel_only():
            with torch.cuda.stream(a):
                for i in range(ITERS):
                    x.add_(1.0)
        res["kernel_only"] = timed(dev, [a], kernel_only)

    if torch.cuda.device_count() > 1:
        d1 = torch.device("cuda:1")
        torch.cuda.set_device(dev)
        torch.empty(1, device=dev).copy_(torch.empty(1, device=d1))  # torch enables peer access
        torch.cuda.set_device(d1)
        torch.empty(1, device=d1).copy_(torch.empty(1, device=dev))
        c = torch.cuda.Stream(d1)
        torch.cuda.set_device(dev)
        g0 = torch.zeros(8, dtype=torch.int32, device=dev)
        g1 = torch.zeros(8, dtype=torch.int32, device=d1)
        for name, fl in ((tag, None),):
            g0.zero_(); g1.zero_()
            torch.cuda.synchronize(d1)

            def remote_write_chain():
                for i in range(ITERS):
                    write(a, ptr(g1), i + 1, fl)
            res[f"peer_write_chain_{name}"] = timed(dev, [a], remote_write_chain)
            g0.zero_(); g1.zero_()
            torch.cuda.synchronize(d1)

            def xgpu_pingpong():
                # GPU0 writes into GPU1's flag, GPU1 (stream c) waits on its local flag and
                # answers into GPU0's memory: the relay's hop pattern
                for i in range(ITERS):
                    write(a, ptr(g1), i + 1, fl)
                    wait(c, ptr(g1), i + 1)
                    write(c, ptr(g0), i + 1, fl)
                    wait(a, ptr(g0), i + 1)
            torch.cuda.synchronize(d1)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(a)
            xgpu_pingpong()
            e1.record(a)
            torch.cuda.synchronize(dev); torch.cuda.synchronize(d1)
            res[f"peer_pingpong_{name}"] = e0.elapsed_time(e1) * 1000.0 / ITERS
    for k, v in res.items():
        print(f"{k:40s} {v:8.2f} us/iter")


if __name__ == "__main__":
    main()
