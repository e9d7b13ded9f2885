"""Decode-attention benchmark (BASELINE.json metric: decode-attention KV GB/s, fraction of the
HBM roofline, attention tokens/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A step is one decode iteration of the workload over every layer: per layer, append each
request's new-token K/V into the paged HBM store and run decode attention over the full
context — one fused lam_decode launch (k_new/v_new), or lam_kv_append + lam_decode with
--separate-append.  KV bytes are the reference's algorithmic bytes
(attn_cost, reference core/src/perf.cpp:77-88): 2 e (d/G) L l B per step.

Default workload (N=1): BASELINE config 2, LLaMA-2-7B all 32 layers, bf16, B=64, l=4096 —
137 GB of KV resident in HBM (far above the 126 MB L2, so no flush is needed).
With N>1 (torchrun, one rank per GPU) the KV heads are sharded over ranks
(head_partition, attention.cpp:164-177).  --scaling strong (the default for N>1) keeps the
workload's global batch fixed — each rank is the model worker of B/N requests and the attention
worker of Hkv/N heads of all B requests, so T1/(N*TN) is the parallel efficiency of BASELINE.md
§3 — and --scaling weak gives every rank B requests (global batch N*B).  Q/K/V reach the head
owners and outputs return over NVLink peer memory (or NCCL all-to-all with --transport nccl),
overlapped with attention across two staggered micro-batches.

After the timed regions the bench checks its own outputs (--check 1, the default): on seeded
(request, q head) pairs of three layers, the output of the benchmarked launch configuration
against the CPU oracle (oracle/, the restatement of attention.cpp:48-70) on the same pool
contents, within the north-star bound, and the fused append bit-exact.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "decode-attention KV GB/s"

# workload -> shape (BASELINE.json configs)
WORKLOADS = {
    "c1": dict(desc="LLaMA-7B 1 layer MHA fp32 B=8 l=1024 (dense, as the CPU reference runs it)",
               spec="LLAMA_7B_1L_F32", B=8, l=1024, Hq=32, Hkv=32, D=128, layers=1,
               dtype="float32", paged=False, P=64),
    "c2": dict(desc="LLaMA-2-7B 32 layers MHA bf16 B=64 l=4096 paged", spec="LLAMA2_7B", B=64,
               l=4096, Hq=32, Hkv=32, D=128, layers=32, dtype="bfloat16", paged=True, P=64),
    "c3": dict(desc="LLaMA-2-70B GQA 64/8 bf16 B=128 l=4096 paged", spec="LLAMA2_70B", B=128,
               l=4096, Hq=64, Hkv=8, D=128, layers=80, dtype="bfloat16", paged=True, P=64),
    "c4": dict(desc="LLaMA-2-70B GQA 64/8 bf16 B=32 l=32768 paged, split-K", spec="LLAMA2_70B",
               B=32, l=32768, Hq=64, Hkv=8, D=128, layers=80, dtype="bfloat16", paged=True, P=64),
    "c5": dict(desc="LLaMA-2-70B GQA mixed lengths 128..16384 (log-uniform, seed 2024) B=256 paged",
               spec="LLAMA2_70B", B=256, l=16384, Hq=64, Hkv=8, D=128, layers=80,
               dtype="bfloat16", paged=True, P=64, mixed=True),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks sampling
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, p in zip(names, parts[4:8]):
                if p.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(sm),
                "reasons": sorted(reasons)}


def ncu_traffic(workload: str, world: int, launch: str, kernel: str):
    """DRAM bytes per decode launch from the committed ncu capture of this workload's launch
    (profiles/ncu_traffic.json, keyed workload/launch/kernel), or None when no capture of this
    launch shape exists."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        d = json.loads(p.read_text()).get(f"{workload}/{launch}/{kernel}")
    except Exception:
        return None
    return d["traffic"] if d and world == 1 else None


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


# ---------------------------------------------------------------- CPU baseline
def cpu_baseline(w: dict, target_s: float, seed: int = 1) -> dict:
    """The reference's own exact_attention<float> (oracle/_ref, built from
    reference core/src/attention.cpp -O3) over a bounded sample of the workload's
    (request, kv head) units, all host threads; falls back to our C port (1 thread)."""
    import numpy as np

    from oracle import oracle as O
    from paper_2405_01814_b200 import perf as PF

    spec = getattr(PF, w["spec"])
    e = spec.bytes_per_elem
    D, Hq, Hkv, l = w["D"], w["Hq"], w["Hkv"], w["l"]
    G = Hq // Hkv
    rng = np.random.default_rng(seed)
    hw = os.cpu_count() or 1
    unit_bytes = 2 * l * D * 4
    units = int(max(8, min(4 * hw, (2 * 2**30) // unit_bytes)))
    B = max(1, -(-units // Hkv))
    units = B * Hkv
    q = rng.uniform(-1, 1, (B, Hq, D)).astype(np.float32)
    k = rng.uniform(-1, 1, (B, Hkv, l, D)).astype(np.float32)
    v = rng.uniform(-1, 1, (B, Hkv, l, D)).astype(np.float32)
    lens = np.full(B, l, np.int32)
    bytes_per_run = units * l * 2 * D * e  # algorithmic bytes in the workload's dtype
    if O.ref_available():
        lib = O.ref()
        threads = int(lib.ref_hardware_threads()) or os.cpu_count() or 1
        h = lib.ref_bench_create(B, Hq, Hkv, D, l, O.ptr(lens), O.ptr(q), O.ptr(k), O.ptr(v),
                                 1.0 / math.sqrt(D), units)
        lib.ref_bench_run(h, threads, None)  # warm
        runs, secs = 0, 0.0
        while runs == 0 or secs < target_s:
            secs += lib.ref_bench_run(h, threads, None)
            runs += 1
        lib.ref_bench_destroy(h)
        kind = "reference"
    else:
        threads = 1
        runs, secs = 0, 0.0
        while runs == 0 or secs < target_s:
            t0 = time.perf_counter()
            O.decode_dense(q, k, v, lens, 1.0 / math.sqrt(D))
            secs += time.perf_counter() - t0
            runs += 1
        kind = "port"
    gbs = bytes_per_run * runs / secs / 1e9
    cpu_model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu_model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"value": gbs, "unit": "GB/s", "cores": threads, "kind": kind,
            "seconds": secs, "runs": runs,
            "sample": (f"{units} (request, kv head) units x {G} q heads x l={l}, d={D} of one "
                       f"layer, exact_attention<float> on fp32 upcasts, {runs} runs, "
                       f"{threads} threads; bytes = attn_cost with e={e}"),
            "cpu_model": cpu_model,
            "attn_tokens_per_s_equiv": gbs * 1e9 / (PF.kv_bytes_per_token(spec) * l)}


def run_reference(args, w: dict, rank: int, world: int) -> None:
    if rank != 0:
        return
    from paper_2405_01814_b200 import perf as PF

    spec = getattr(PF, w["spec"])
    for _ in range(args.warmup):
        cpu_baseline(w, target_s=0.0)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        r = cpu_baseline(w, target_s=0.5)
        vals.append(r["value"])
        secs += r["seconds"]
    value = statistics.median(vals)
    step_bytes = PF.attn_cost(spec, w["B"], w["l"]).bytes
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_bytes / (value * 1e9) * 1e3,
            "ms_per_step_basis": ("extrapolated: the step's attn_cost bytes / the rate measured on "
                                  "the bounded sample (one layer, a subset of units); not timed "
                                  "over a whole step"),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic U(-1,1)",
            "config": {"workload": f"{args.workload}: {w['desc']}",
                       "global_batch": w["B"] * (world if args.scaling == "weak" else 1),
                       "seq_len": w["l"], "layers": w["layers"],
                       "parallelism": "host threads"},
            "attn_tokens_per_s": value * 1e9 / (PF.kv_bytes_per_token(spec) * w["l"]),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": r["cores"],
                             "kind": r["kind"], "sample": r["sample"], "cpu_model": r["cpu_model"]},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU workload
def mixed_lengths(B: int, seed: int = 2024):
    import numpy as np

    r = np.random.default_rng(seed)
    return np.exp(r.uniform(math.log(128), math.log(16384), B)).astype(np.int32)


class Workload:
    """Resident paged KV for every layer (or as many distinct layer buffers as fit) plus
    per-layer new-token inputs; one GPU's share under KV-head sharding."""

    def __init__(self, w: dict, rank: int, world: int, device, engine: bool = False,
                 strong: bool = False, micro_batches: int = 2):
        import numpy as np
        import torch

        from paper_2405_01814_b200 import _lib, perf as PF
        from paper_2405_01814_b200.kvcache import PagedKVCache

        self.w, self.rank, self.world, self.device = w, rank, world, device
        self.spec = getattr(PF, w["spec"])
        self.dtype = getattr(torch, w["dtype"])
        self.Hq, self.Hkv, self.D = w["Hq"], w["Hkv"], w["D"]
        if self.Hkv % world:
            raise SystemExit(f"{self.Hkv} KV heads do not shard over {world} GPUs")
        self.hq_local, self.hkv_local = self.Hq // world, self.Hkv // world
        # requests whose q/k/v this rank produces: a share of the fixed global batch (strong
        # scaling) or a full batch per rank (weak scaling)
        from paper_2405_01814_b200.dist import local_batch

        try:
            self.B_local = local_batch(w["B"], world, "strong" if strong else "weak",
                                       micro_batches if (engine or world > 1) else 1)
        except ValueError as e:
            raise SystemExit(str(e))
        self.B = self.B_local * world         # requests whose local heads this rank attends
        self.layers = w["layers"]
        # the attention-worker engine (always for N > 1): staggered micro-batches (two by default,
        # the paper's schedule)
        engine = engine or world > 1
        self.mb = micro_batches if engine else 1
        self.geo = None
        if engine:
            from paper_2405_01814_b200.dist import ShardGeometry

            self.geo = ShardGeometry(rank, world, self.layers, self.B_local, self.Hq, self.Hkv,
                                     self.D, self.mb)
        # per-source request lengths; attention-side rows are micro-batch major.  Strong scaling
        # deals one global draw out to the sources (the same requests at every N).
        if w.get("mixed") and strong:
            glob = mixed_lengths(self.B, 2024)
            src_lens = [glob[r * self.B_local:(r + 1) * self.B_local] for r in range(world)]
        else:
            src_lens = [mixed_lengths(w["B"], 2024 + r) if w.get("mixed")
                        else np.full(w["B"], w["l"], np.int32) for r in range(world)]
        self.lens = np.zeros(self.B, np.int32)
        for src in range(world):
            for b in range(self.B_local):
                row = self.geo.kv_row(src, b) if self.geo else b
                self.lens[row] = src_lens[src][b]
        self.B_launch = self.B // self.mb
        self.max_len = int(self.lens.max())
        esz = torch.tensor([], dtype=self.dtype).element_size()
        P = w["P"]
        pages_per_seq = -(-self.lens // P)
        self.num_pages = int(pages_per_seq.sum())
        layer_bytes = 2 * self.num_pages * self.hkv_local * P * self.D * esz
        free, _ = torch.cuda.mem_get_info(device)
        budget = free - 6 * 2**30
        # Small workloads rotate over enough distinct buffer sets (>= 1 GiB total) that
        # consecutive steps never find their KV in the 126 MB L2.
        want = max(self.layers, -(-2**30 // layer_bytes))
        self.resident = int(max(1, min(want, budget // layer_bytes)))
        if os.environ.get("LAM_BENCH_RESIDENT"):  # experiments: fewer distinct pool layers
            self.resident = min(self.resident, int(os.environ["LAM_BENCH_RESIDENT"]))
        self.kv_bytes_layer = layer_bytes
        self.ctx = _lib.context(device.index)
        if w["paged"]:
            self.cache = PagedKVCache(self.resident, self.hkv_local, self.D, P, self.num_pages,
                                      self.B, int(pages_per_seq.max()), dtype=self.dtype,
                                      device=device, shuffle_seed=1234 + rank)
            self.cache.set_lengths(self.lens)
            self.cache.sync()
            g = torch.Generator(device=device).manual_seed(1 + rank)
            self.cache.fill_random(g)
            self.k_layers = [self.cache.k[i] for i in range(self.resident)]
            self.v_layers = [self.cache.v[i] for i in range(self.resident)]
            self.page_table = self.cache.page_table
        else:
            g = torch.Generator(device=device).manual_seed(1 + rank)
            shape = (self.B, self.hkv_local, self.max_len, self.D)
            self.k_layers = [torch.empty(shape, dtype=self.dtype, device=device).uniform_(-1, 1, generator=g)
                             for _ in range(self.resident)]
            self.v_layers = [torch.empty(shape, dtype=self.dtype, device=device).uniform_(-1, 1, generator=g)
                             for _ in range(self.resident)]
            self.page_table = None
        self.seq_lens = torch.tensor(self.lens, dtype=torch.int32, device=device)
        self.positions = (self.seq_lens - 1).contiguous()
        # mixed lengths: claim work longest-first (LPT), per launch
        from paper_2405_01814_b200.decode import longest_first

        self.orders = ([longest_first(self.seq_lens[m * self.B // self.mb:(m + 1) * self.B // self.mb])
                        for m in range(self.mb)] if w.get("mixed") else [None] * self.mb)
        gi = torch.Generator(device=device).manual_seed(99 + rank)
        # model-worker side inputs for this rank's B_local requests, per layer
        if self.geo is None:
            qs = (self.layers, self.B_local, self.Hq, self.D)
            ks = (self.layers, self.B_local, self.Hkv, self.D)
            self.q_in = torch.empty(qs, dtype=self.dtype, device=device).uniform_(-1, 1, generator=gi)
            self.kn_in = torch.empty(ks, dtype=self.dtype, device=device).uniform_(-1, 1, generator=gi)
            self.vn_in = torch.empty_like(self.kn_in).uniform_(-1, 1, generator=gi)
        else:
            qs = self.geo.q_shape()
            # packed QKV projection rows per destination shard (one all-to-all per micro-batch)
            self.qkv_in = torch.empty(self.geo.qkv_shape(), dtype=self.dtype,
                                      device=device).uniform_(-1, 1, generator=gi)
        self.out = torch.empty(qs, dtype=self.dtype, device=device)
        # reference attn_cost bytes of one step over ALL requests and heads (whole job)
        self.step_bytes = float(PF.kv_bytes_per_token(self.spec)) * float(self.lens.sum())
        # this rank's algorithmic bytes per decode launch (its KV heads, one micro-batch)
        self.decode_bytes_per_launch = (float(self.lens.sum()) * 2 * self.hkv_local * self.D *
                                        esz / self.mb)
        # plan once (fixed shapes): kernel family + splits; reserve the split-K workspace
        from paper_2405_01814_b200 import decode as dec

        qd = torch.empty((self.B_launch, self.hq_local, self.D), dtype=self.dtype, device=device)
        # split_tokens of every launch: 0 = the library's planner decides (the default)
        self.split_arg = int(os.environ.get("LAM_BENCH_SPLIT_TOKENS", 0))
        kw = dict(page_table=self.page_table[: self.B_launch] if self.page_table is not None
                  else None, max_len=self.max_len)
        self.kernel, self.splits, self.chunk = dec.plan(
            qd, self.k_layers[0], self.v_layers[0], self.seq_lens[: self.B_launch], ctx=self.ctx,
            split_tokens=self.split_arg, **kw)
        self.ctx.reserve(self.B_launch * self.hq_local * max(self.splits, 1), self.D,
                         self.B_launch * self.hkv_local)

    def rows(self, m: int):
        return slice(m * self.B_launch, (m + 1) * self.B_launch)

    def layer_pools(self, layer: int, step: int = 0):
        i = (step * self.layers + layer) % self.resident
        return self.k_layers[i], self.v_layers[i]


def check_outputs(W, engine, step_fn, counter, layers_hint=None, pairs_per_layer=4, seed=7):
    """Checker, outside every timed region: run one more step of the benchmarked launch
    configuration and compare its outputs on seeded (request, q head) pairs of three layers with
    the CPU oracle (exact_attention<float> restated, attention.cpp:48-70, on the exactly upcast
    pool contents) — max-abs within the north-star bound — and the fused append bit-exact (the
    pool row at seq_len - 1 equals the new token).  Each rank checks the rows it both produced
    (model worker) and attended (attention worker).  Returns (max_abs_err, n_pairs, append_ok)."""
    import numpy as np
    import torch

    from oracle import oracle as O

    s = counter[0]
    step_fn()
    torch.cuda.synchronize(W.device)
    rng = np.random.default_rng(seed + W.rank)
    L = W.layers
    # with fewer resident pool sets than layers, layers l and l + resident share a pool within a
    # step and the later one's append is what the pool holds: check layers no later layer aliases
    lo = max(0, L - W.resident)
    layers = sorted({lo, min(lo + 1, L - 1), L - 1} if layers_hint is None else set(layers_hint))
    G = W.Hq // W.Hkv
    scale = 1.0 / math.sqrt(W.D)
    P = W.w["P"]
    worst, n, append_ok = 0.0, 0, True
    for layer in layers:
        if engine is None:  # plain per-layer launches: rows are requests, all heads local
            kp, vp = W.layer_pools(layer, s)
            cand = [(b, b) for b in range(W.B)]
        else:  # engine: this rank's own requests, its own head shard
            kp, vp = W.layer_pools(layer)
            g = W.geo
            cand = [(g.kv_row(W.rank, bl), bl) for bl in range(W.B_local)]
        for _ in range(pairs_per_layer):
            row, bl = cand[int(rng.integers(len(cand)))]
            h = int(rng.integers(W.hq_local))
            kvh = h // G
            ln = int(W.lens[row])
            if engine is None:
                q = W.q_in[layer, bl, h]
                k_new, v_new = W.kn_in[layer, bl, kvh], W.vn_in[layer, bl, kvh]
                out = W.out[layer, bl, h]
            else:
                m, i = divmod(bl, g.Bh)
                rows = W.qkv_in[layer, m, W.rank, i]
                q, k_new, v_new = rows[h], rows[g.hq_l + kvh], rows[g.hq_l + g.hkv_l + kvh]
                out = W.out[layer, m, W.rank, i, h]
            if W.page_table is not None:
                npg = -(-ln // P)
                pages = W.page_table[row, :npg].long()
                kd = kp[pages, kvh].reshape(-1, W.D)[:ln]
                vd = vp[pages, kvh].reshape(-1, W.D)[:ln]
            else:
                kd, vd = kp[row, kvh, :ln], vp[row, kvh, :ln]
            append_ok &= bool(torch.equal(kd[ln - 1], k_new) and torch.equal(vd[ln - 1], v_new))
            want = O.decode_dense(q.float().cpu().numpy()[None, None], kd.float().cpu().numpy()[None, None],
                                  vd.float().cpu().numpy()[None, None], np.array([ln], np.int32), scale)
            err = float(np.abs(out.float().cpu().numpy() - want[0, 0]).max())
            worst, n = max(worst, err), n + 1
    return worst, n, append_ok


def run_ours(args, w: dict, rank: int, world: int) -> None:
    import numpy as np
    import torch

    from paper_2405_01814_b200 import _lib, decode as dec

    device = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=device)
    t_setup = time.time()
    use_engine = world > 1 or args.engine == "peer"
    if world == 1 and use_engine and args.transport != "peer":  # (NCCL needs N > 1)
        raise SystemExit("--engine peer at one GPU needs --transport peer")
    strong = args.scaling == "strong"
    W = Workload(w, rank, world, device, engine=use_engine, strong=strong,
                 micro_batches=args.micro_batches)
    if args.overlap_layers is None:
        # consecutive launches of a step are different layers (their pools are disjoint) only
        # when the model has more than one layer; a one-layer stream would have each launch
        # read the rows its predecessor appended, which overlap_prev's contract excludes
        args.overlap_layers = int(W.layers >= 2 and engine_is_local(args, world))
    log(f"[rank {rank}] setup {time.time() - t_setup:.1f}s: {W.resident}/{W.layers} layers resident, "
        f"kernel={W.kernel} splits={W.splits} chunk={W.chunk}")

    stream = torch.cuda.current_stream(device)
    # one persistent launch per step: for multi-layer paged workloads (one-layer C1 has no layer
    # boundary to remove)
    use_step = (args.launch == "step" and not args.separate_append and W.layers > 1
                and W.page_table is not None)
    engine = None
    if use_engine:
        from paper_2405_01814_b200.dist import HeadShardedAttention

        def attend(layer, m, q, k, v, out):  # fused append + decode, straight from the
            kp, vp = W.layer_pools(layer)      # packed receive buffer
            sl = W.rows(m)
            dec.decode(q, kp, vp, W.seq_lens[sl],
                       page_table=W.page_table[sl] if W.page_table is not None else None,
                       max_len=W.max_len, out=out, ctx=W.ctx, split_tokens=W.split_arg,
                       k_new=k, v_new=v, request_order=W.orders[m])

        if args.transport == "peer":
            from paper_2405_01814_b200.dist import PeerShardedAttention

            def launch_args(layer, m):
                kp, vp = W.layer_pools(layer)
                sl = W.rows(m)
                g = W.geo
                qd = torch.empty((g.B_mb, g.hq_l, g.D), dtype=W.dtype, device=device)
                a, _ = dec.make_args(qd, kp, vp, W.seq_lens[sl],
                                     page_table=W.page_table[sl] if W.page_table is not None else None,
                                     max_len=W.max_len, out=qd, split_tokens=W.split_arg,
                                     request_order=W.orders[m])
                return a

            def step_args():  # the step launch: every attention row, pool layer 0
                kp, vp = W.layer_pools(0)
                qd = torch.empty((W.B, W.geo.hq_l, W.D), dtype=W.dtype, device=device)
                a, _ = dec.make_args(qd, kp, vp, W.seq_lens, page_table=W.page_table,
                                     max_len=W.max_len, out=qd)
                if W.orders[0] is not None:
                    W.order_all = torch.cat(W.orders).contiguous()
                    a.request_order = W.order_all.data_ptr()
                return a, W.resident, kp.numel() // W.D

            sync = os.environ.get("LAM_PEER_SYNC", "step" if use_step else "kernel")
            engine = PeerShardedAttention(W.geo, dist, W.ctx, launch_args, device, W.dtype,
                                          sync=sync, step_args=step_args,
                                          relay=args.relay if sync == "step" else "stream")
            engine.qkv_in.copy_(W.qkv_in)
            W.qkv_in = engine.qkv_in
            W.out = engine.out
        else:
            engine = HeadShardedAttention(W.geo, dist, None, attend, device, W.dtype)

    counter = [0]
    arg_cache = {}
    lib, sp = _lib.load(), stream.cuda_stream

    def step_local(ev=None):
        """world == 1: append + decode per layer on the current stream (or all layers in one
        step launch)."""
        s = counter[0]
        counter[0] += 1
        if use_step:
            if ev is not None:
                ev[0][0].record(stream)
            dec.decode_step(W.q_in, W.cache.k, W.cache.v, W.seq_lens, page_table=W.page_table, max_len=W.max_len, out=W.out,
                            k_new=W.kn_in, v_new=W.vn_in, request_order=W.orders[0],
                            layer0=(s * W.layers) % W.resident, ctx=W.ctx)
            if ev is not None:
                ev[0][1].record(stream)
            return
        for layer in range(W.layers):
            kp, vp = W.layer_pools(layer, s)
            if ev is not None:
                ev[layer][0].record(stream)
            if args.separate_append:
                dec.kv_append(W.kn_in[layer], W.vn_in[layer], kp, vp, W.positions, W.page_table)
                dec.decode(W.q_in[layer], kp, vp, W.seq_lens, page_table=W.page_table,
                           max_len=W.max_len, out=W.out[layer], ctx=W.ctx, split_tokens=W.split_arg)
            else:  # one launch: append the new token and attend (fused lam_kv_append)
                key = (layer, (s * W.layers + layer) % W.resident)
                a = arg_cache.get(key)
                if a is None:  # lam_decode_args built once per (layer, pool set)
                    a, _ = dec.make_args(W.q_in[layer], kp, vp, W.seq_lens,
                                         page_table=W.page_table, max_len=W.max_len,
                                         out=W.out[layer], split_tokens=W.split_arg,
                                         k_new=W.kn_in[layer], v_new=W.vn_in[layer],
                                         request_order=W.orders[0],
                                         overlap_prev=args.overlap_layers)
                    arg_cache[key] = a
                _lib.check(lib.lam_decode(W.ctx.handle, a, sp))
            if ev is not None:
                ev[layer][1].record(stream)

    def step(ev=None):
        if engine is None:
            step_local(ev)
        elif args.transport == "peer":
            engine.step(ev)
        else:
            engine.step(W.qkv_in, W.out, ev)

    def barrier():
        torch.cuda.synchronize(device)
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize(device)

    # ---- warm-up
    for i in range(max(args.warmup, 0)):
        tw = time.time()
        step()
        if os.environ.get("LAM_BENCH_VERBOSE"):
            torch.cuda.synchronize(device)
            log(f"[rank {rank}] warm-up step {i}: {1e3 * (time.time() - tw):.1f} ms, "
                f"status {W.ctx.status(clear=False)}")
    barrier()

    # ---- timed region (device-resident inputs)
    # Self-synchronising peer launches overlap their neighbours (programmatic dependent launch);
    # an event between two launches would serialise them, so the timed region then carries
    # only the step events and a launch's duration is the step time / launches (an upper bound).
    step_launch = use_step and (engine is None or (args.transport == "peer" and engine.sync == "step"))
    n_launch = 1 if step_launch else W.layers * W.mb  # decode launches per step and rank
    pdl = engine is not None and args.transport == "peer" and engine.sync == "kernel" and \
        os.environ.get("LAM_PDL", "1") != "0"
    pdl = pdl or (engine is None and args.overlap_layers and not args.separate_append)
    pdl = pdl and not step_launch
    # The timed region carries no per-launch events (an event between two launches adds a gap
    # on the stream: C1's 51 us launches lost 6 %); the decode kernel's own duration is timed by
    # an instrumented pass over the same steps right after (non-PDL modes).
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(device.index if "CUDA_VISIBLE_DEVICES" not in os.environ else
                           int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[device.index]))
    if rank == 0:
        sampler.start()
        time.sleep(0.3)
    barrier()
    # one untimed step is already in flight when the first event is recorded, so the host has
    # queued the timed steps before the GPU reaches them (C1's 48 us launches would otherwise
    # count the Python call that enqueues the first one)
    step(None)
    t0.record(stream)
    for s in range(args.steps):
        step(None)
    t1.record(stream)
    barrier()
    clocks = sampler.stop() if rank == 0 else None
    ms_total = t0.elapsed_time(t1)
    ms_step = ms_total / max(args.steps, 1)
    one_launch = n_launch == 1 and not args.separate_append
    if step_launch or one_launch:  # the launch is the step (its time bounds the launch's)
        kern_ms = [ms_step]
    elif pdl:
        kern_ms = [ms_step / (W.layers * W.mb)]
    else:  # instrumented pass: CUDA events around every decode launch, same steps
        ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)]
               for _ in range(W.layers * W.mb)] for _ in range(args.steps)]
        barrier()
        for s in range(args.steps):
            step(ev[s])
        barrier()
        kern_ms = [e[0].elapsed_time(e[1]) for s in range(args.steps) for e in ev[s]]
    if dist is not None:
        t = torch.tensor([ms_step, statistics.mean(kern_ms)], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step, kern_avg = float(t[0]), float(t[1])
    else:
        kern_avg = statistics.mean(kern_ms)
    launches = args.steps * n_launch * (2 if args.separate_append else 1)
    alone_ms = None
    if pdl:
        # diagnostic: the same step with launches serialised and timed one by one
        os.environ["LAM_PDL"] = "0"
        ev1 = [[torch.cuda.Event(enable_timing=True) for _ in range(2)]
               for _ in range(W.layers * W.mb)]
        barrier()
        step(ev1)
        barrier()
        os.environ["LAM_PDL"] = "1"
        alone_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev1)
    if engine is not None and args.transport != "peer":
        # the same decode launch with no collective in flight (diagnoses comm interference)
        g = W.geo
        packed = engine.qkv_r[0].view(g.B_mb, g.W, g.D)
        sl = W.rows(0)
        kp, vp = W.layer_pools(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        torch.cuda.synchronize(device)
        e0.record(stream)
        for _ in range(reps):
            dec.decode(packed[:, : g.hq_l], kp, vp, W.seq_lens[sl],
                       page_table=W.page_table[sl] if W.page_table is not None else None,
                       max_len=W.max_len, out=engine.o_l[0].view(g.B_mb, g.hq_l, g.D), ctx=W.ctx,
                       split_tokens=W.split_arg, request_order=W.orders[0])
        e1.record(stream)
        torch.cuda.synchronize(device)
        alone_ms = e0.elapsed_time(e1) / reps

    tdir = os.environ.get("LAM_STEP_TRACE")  # diagnostic: the last timed step's stamps
    if tdir and getattr(engine, "trace_buf", None) is not None:
        torch.cuda.synchronize(device)
        os.makedirs(tdir, exist_ok=True)
        np.save(os.path.join(tdir, f"rank{rank}.npy"), engine.trace_buf.cpu().numpy())

    # ---- end-to-end through the C-ABI host-buffer entry point (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, W, engine, dist, device, stream, use_step)

    # ---- output check of the benchmarked launch configuration (outside the timed regions)
    check = None
    if args.check:
        tol = {"bfloat16": 2e-3, "float16": 2e-3, "float32": 1e-5}[w["dtype"]]
        if w["dtype"] != "float32" and W.out.dtype != torch.float32:
            tol += 2.0 ** -9  # the bench's outputs are stored in bf16 (|out| < 1)
        err, n, app = check_outputs(W, engine, step, counter)
        t = torch.tensor([err, float(not app)], device=device, dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        err, app = float(t[0]), not bool(t[1])
        check = {"checker": "CPU oracle (oracle/: exact_attention<float> restated, attention.cpp:48-70) on the "
                            "upcast pool contents after one more step; outside the timed regions",
                 "pairs_per_rank": n, "max_abs": err, "tol": tol, "append_bit_exact": app,
                 "ok": bool(err <= tol and app)}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    peaks = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    value = W.step_bytes / (ms_step / 1e3) / 1e9
    bytes_per_launch = W.decode_bytes_per_launch * W.layers * W.mb / n_launch
    achieved = bytes_per_launch / (kern_avg / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": {"bfloat16": "bf16", "float32": "f32", "float16": "f16"}[w["dtype"]],
        "data": "synthetic: q, k, v ~ U(-1,1) (bench_attention.cpp:11-27 law), shuffled page placement",
        "config": {"workload": f"{args.workload}: {w['desc']}", "global_batch": W.B,
                   "seq_len": int(W.max_len), "sum_seq_len": int(W.lens.sum()) ,
                   "layers": W.layers, "kv_layers_resident": W.resident,
                   "q_heads": W.Hq, "kv_heads": W.Hkv, "head_dim": W.D, "page_size": w["P"],
                   "parallelism": (f"kv-head sharded x{world} ({args.transport})" if world > 1 else
                                   "single GPU" + (", attention-worker engine (2 micro-batches, peer transport)"
                                                   if use_engine else "")),
                   "l2": f"inputs {W.kv_bytes_layer * W.resident / 2**30:.0f} GiB of KV >> 126 MB L2; no flush needed",
                   "timed_region": "K back-to-back steps; one untimed step is in flight when the first event is recorded",
                   "kernel": W.kernel,
                   "splits": ("lam_decode_step's choice (S = 1 without input waits; with them, "
                              "items of at most 8 K tokens)") if step_launch else W.splits,
                   "split_tokens": None if step_launch else W.chunk,
                   "launch": "step" if step_launch else "per layer and micro-batch",
                   "micro_batches": W.mb,
                   "overlap_layers": bool(args.overlap_layers) and not step_launch,
                   **({"model_worker": ("zero-compute stand-in: layer l+1 inputs follow layer l "
                                        "outputs of all ranks, relayed "
                                        + ("inside the step launch (lam_peer_io.n_relay)"
                                           if getattr(engine, "relay", "") == "kernel" and use_step
                                           else "by stream memory operations"))}
                      if world > 1 and args.transport == "peer" else {})},
        "attn_tokens_per_s": W.B / (ms_step / 1e3),
        "frac_of_hbm_roofline": value / world / peak,
        "frac_of_hbm_spec_8tbs": value / world / 8000.0,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650",
                     "kernel": f"decode_{W.kernel}", "bytes_per_launch": bytes_per_launch,
                     "avg_launch_ms": kern_avg, "traffic": ncu_traffic(args.workload, world, "step" if step_launch else "layer", W.kernel),
                     "launch_timing": ("one persistent launch per step (lam_decode_step): the launch "
                                       "is the step" if step_launch else
                                       "one launch per step: the step time (an upper bound of "
                                       "the launch's duration)" if one_launch else
                                       "step time / launches (back-to-back launches overlap under "
                                       "programmatic dependent launch)" if pdl else
                                       "CUDA events around every launch, in an instrumented "
                                       "pass over the same steps right after the timed region"),
                     "alone_launch_ms": alone_ms},
        "gpu_launches": launches,
        "device_status": W.ctx.status(clear=False),  # LAM_STATUS_* (0: no bounded wait expired)
        "clocks": clocks,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if check is not None:
        line["check"] = check
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(w, target_s=args.cpu_seconds)
        except Exception as exc:  # the CPU baseline is reported, never required
            line["cpu_baseline"] = {"error": repr(exc)}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    if check is not None and not check["ok"]:
        raise SystemExit("output check FAILED: the numbers above are not valid")


def engine_is_local(args, world: int) -> bool:
    """plain per-layer launches on one GPU (no attention-worker engine)"""
    return world == 1 and args.engine == "local" and not args.separate_append


def run_e2e(args, W, engine, dist, device, stream, use_step=False):
    """Same step from host memory through the C-ABI (lam_decode_step_from_host for step launches,
    else lam_decode_layers_host): every layer's q / k_new / v_new copied from pinned host memory
    and its output copied back, inside the timed region; copies overlap the HBM-bound
    attention."""
    import ctypes as C

    import torch

    from paper_2405_01814_b200 import _lib, decode as dec

    lib = _lib.load()
    L = W.layers
    h_out = torch.empty(W.out.shape, dtype=W.out.dtype).pin_memory()
    if engine is not None:
        h_qkv = W.qkv_in.cpu().pin_memory()

        def step_mg():
            if args.transport == "peer":
                engine.step(host_in=h_qkv, host_out=h_out)
            else:
                engine.step(W.qkv_in, W.out, host_in=h_qkv, host_out=h_out)

        for _ in range(max(1, args.warmup)):
            step_mg()
        torch.cuda.synchronize(device)
        if dist is not None:
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step_mg()
        t1.record(stream)
        torch.cuda.synchronize(device)
        t = torch.tensor([t0.elapsed_time(t1) / max(args.steps, 1)], device=device)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        h2d = h_qkv.numel() * h_qkv.element_size()
        d2h = h_out.numel() * h_out.element_size()
        return {"value": W.step_bytes / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
                "h2d_bytes_per_step": int(h2d) * W.world, "d2h_bytes_per_step": int(d2h) * W.world,
                "api": ("PeerShardedAttention.step (pinned host in/out overlapped on copy streams, "
                        "zero-copy NVLink peer transport)" if args.transport == "peer" else
                        "HeadShardedAttention.step (pinned host in/out overlapped on copy streams, "
                        "NCCL all-to-all)")}
    h_q = W.q_in.cpu().pin_memory()
    h_kn = W.kn_in.cpu().pin_memory()
    h_vn = W.vn_in.cpu().pin_memory()
    d_q = torch.empty_like(W.q_in[0])
    d_out = torch.empty_like(W.out[0])
    if use_step:
        return run_e2e_step(args, W, device, stream, h_q, h_kn, h_vn, h_out, d_q, d_out)
    # per-layer argument blocks (pools rotate like the device-resident loop)
    ArgsArr = dec.DecodeArgs * L
    args_sets = []
    for s in range(max(1, W.resident // L if W.resident >= L else 1)):
        arr = ArgsArr()
        for layer in range(L):
            kp, vp = W.layer_pools(layer, s)
            a, _ = dec.make_args(d_q, kp, vp, W.seq_lens, page_table=W.page_table,
                                 max_len=W.max_len, out=d_out, split_tokens=W.split_arg,
                                 request_order=W.orders[0])
            arr[layer] = a
        args_sets.append(arr)
    stage = torch.empty(int(lib.lam_decode_layers_host_stage_bytes(args_sets[0])),
                        dtype=torch.uint8, device=device)
    P = C.c_void_p * L
    hq = P(*[h_q[i].data_ptr() for i in range(L)])
    hk = P(*[h_kn[i].data_ptr() for i in range(L)])
    hv = P(*[h_vn[i].data_ptr() for i in range(L)])
    ho = P(*[h_out[i].data_ptr() for i in range(L)])
    copy_stream = torch.cuda.Stream(device=device)
    sp, xp = stream.cuda_stream, copy_stream.cuda_stream
    counter = [0]

    def step():
        s = counter[0] % len(args_sets)
        counter[0] += 1
        _lib.check(lib.lam_decode_layers_host(W.ctx.handle, args_sets[s], L, hq, hk, hv, ho,
                                              stage.data_ptr(), W.positions.data_ptr(), sp, xp))

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize(device)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(device)
    ms = t0.elapsed_time(t1) / max(args.steps, 1)
    # the library takes the zero-copy path for a one-layer step (LAM_HOST_ZERO_COPY overrides)
    zc = os.environ.get("LAM_HOST_ZERO_COPY", "-1")
    zero_copy = zc == "1" or (zc not in ("0", "1") and L == 1)
    h2d = (h_q.numel() + h_kn.numel() + h_vn.numel()) * h_q.element_size()
    d2h = h_out.numel() * h_out.element_size()
    return {"value": W.step_bytes / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": ("lam_decode_layers_host (C-ABI, pinned host buffers, zero-copy: the launch reads "
                    "q / k_new / v_new from and stores the outputs into the mapped host buffers "
                    "over PCIe)" if zero_copy else
                    "lam_decode_layers_host (C-ABI, pinned host buffers, copies overlapped)")}


def run_e2e_step(args, W, device, stream, h_q, h_kn, h_vn, h_out, d_q, d_out):
    """e2e through lam_decode_step_from_host: one step launch that waits per layer for that
    layer's host inputs (in-kernel sequence numbers) while later layers are still being copied,
    and returns each layer's output as soon as it is published."""
    import ctypes as C

    import torch

    from paper_2405_01814_b200 import _lib, decode as dec

    lib = _lib.load()
    L = W.layers
    a, _ = dec.make_args(d_q, W.cache.k[0], W.cache.v[0], W.seq_lens, page_table=W.page_table,
                         max_len=W.max_len, out=d_out, request_order=W.orders[0])
    st = dec.step_layout(L, 1, W.B, pool_layers=W.resident,
                         pool_layer_rows=W.cache.k[0].numel() // W.D)
    stage = torch.empty(int(lib.lam_decode_step_from_host_stage_bytes(a, L)), dtype=torch.uint8,
                        device=device)
    P = C.c_void_p * L
    hq = P(*[h_q[i].data_ptr() for i in range(L)])
    hk = P(*[h_kn[i].data_ptr() for i in range(L)])
    hv = P(*[h_vn[i].data_ptr() for i in range(L)])
    ho = P(*[h_out[i].data_ptr() for i in range(L)])
    copy_stream = torch.cuda.Stream(device=device)
    sp, xp = stream.cuda_stream, copy_stream.cuda_stream
    counter = [0]

    def step():
        st.layer0 = (counter[0] * L) % W.resident
        counter[0] += 1
        _lib.check(lib.lam_decode_step_from_host(W.ctx.handle, a, st, hq, hk, hv, ho,
                                                 stage.data_ptr(), sp, xp))

    for _ in range(max(1, args.warmup)):
        step()
    torch.cuda.synchronize(device)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize(device)
    ms = t0.elapsed_time(t1) / max(args.steps, 1)
    # the library takes the zero-copy path for a one-layer step (LAM_HOST_ZERO_COPY overrides)
    zc = os.environ.get("LAM_HOST_ZERO_COPY", "-1")
    zero_copy = zc == "1" or (zc not in ("0", "1") and L == 1)
    h2d = (h_q.numel() + h_kn.numel() + h_vn.numel()) * h_q.element_size()
    d2h = h_out.numel() * h_out.element_size()
    return {"value": W.step_bytes / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": ("lam_decode_step_from_host (C-ABI, pinned host buffers; one step launch that "
                    "waits in-kernel for each layer's copied inputs, outputs copied back per layer)")}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", 1)))
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU reference sample length for cpu_baseline (seconds of CPU work)")
    ap.add_argument("--transport", default="peer", choices=["nccl", "peer"],
                    help="multi-GPU scatter/gather: NCCL all-to-all or zero-copy NVLink peer memory")
    ap.add_argument("--engine", default="local", choices=["local", "peer"],
                    help="one GPU: plain per-layer launches, or the attention-worker engine of the "
                         "multi-GPU runs (2 micro-batches, self-synchronising launches)")
    ap.add_argument("--overlap-layers", type=int, default=None, choices=[0, 1],
                    help="one GPU: each layer's launch may stream its first KV tiles while the "
                         "previous layer's launch drains (lam_decode_args.overlap_prev; q / k_new "
                         "/ v_new are read only after the previous launch completes).  Default: on "
                         "for multi-layer workloads, off for one layer (c1)")
    ap.add_argument("--separate-append", action="store_true",
                    help="lam_kv_append + lam_decode per layer instead of the fused launch")
    ap.add_argument("--scaling", default=None, choices=["strong", "weak"],
                    help="N>1: fixed global batch (strong, the default) or B requests per rank (weak)")
    ap.add_argument("--micro-batches", type=int, default=2,
                    help="N>1 (and --engine peer): staggered micro-batches of the attention-worker "
                         "engine (the paper's schedule uses two)")
    ap.add_argument("--launch", default="step", choices=["step", "layer"],
                    help="one persistent launch per decode step covering every layer and "
                         "micro-batch (lam_decode_step), or one launch per layer and micro-batch")
    ap.add_argument("--relay", default="stream", choices=["stream", "kernel"],
                    help="N > 1: the zero-compute model worker's layer-to-layer relay: stream "
                         "operations per micro-batch, or forwarded inside the step launch")
    ap.add_argument("--check", type=int, default=1, choices=[0, 1],
                    help="after the timed regions, check the benchmarked launches' outputs against "
                         "the CPU oracle on seeded (request, head) pairs of three layers")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.gpus != world and world == 1 and args.gpus > 1:
        log(f"--gpus {args.gpus} requested without torchrun: running one rank")
        args.gpus = 1
    w = dict(WORKLOADS[args.workload])
    if os.environ.get("LAM_BENCH_SEQ"):  # diagnostic: shorter contexts (relay latency probes)
        w["l"] = int(os.environ["LAM_BENCH_SEQ"])
        w["desc"] += f" [LAM_BENCH_SEQ={w['l']}: diagnostic, not the workload]"
    if args.scaling is None:  # (at N = 1 both mean the same workload)
        args.scaling = "strong"
    if args.impl == "reference":
        run_reference(args, w, rank, world)
    else:
        run_ours(args, w, rank, world)


if __name__ == "__main__":
    main()
