"""Export measured B200 attention numbers in the reference planner's own input formats.

The reference plans deployments analytically: attention time is
roofline_time(attn_cost, memory_pool, EfficiencyProfile, attention) (reference
core/src/sim.cpp:295-301), derated by EfficiencyProfile.attn_mbu (perf.hpp:30-35, default 0.80,
"calibration knobs, not measurements"), and transfers by a NetPreset (net.hpp; FHBN and NCCL-GDR
measured over 400 Gb/s RoCE, net.cpp:13-18).  This script turns bench.py results into:

  * a DISAGG_CATALOG extension file (reference tools/common.cpp:18-40) with a B200 DeviceSpec
    (model.cpp:180-193 schema; it must pass DeviceSpec::validate, model.cpp:72-80 — the price is
    an estimate, labelled as such) and the LLaMA-2 models BASELINE.json names (the reference
    catalog has neither, catalog.cpp:39-53);
  * the measured attention MBU to pass as --attn-mbu (main.cpp:23), and the measured per-layer
    attention time for --ta-ms (main.cpp:38, cmd_analysis.cpp:92-99);
  * an NVLINK-PEER NetPreset measured on the peer transport (experiments/r02/nvlink_preset.py),
    beside the reference's FHBN / NCCL-GDR;
  * the reference's max_batch (perf.cpp:130-140) for B200 attention pools (restated in
    perf.max_batch; tests/test_planner_cpu.py checks both against the reference's own code).

    python scripts/export_catalog.py profiles/r02/bench_c3_n1.json profiles/r02/bench_c2_n1.json \
        profiles/r02/nvlink_preset.json > integration/b200_catalog.json
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2405_01814_b200 import perf as PF  # noqa: E402

# B200 device figures: dense bf16 peak, HBM capacity and bandwidth at spec (the planner derates
# them with the efficiency profile), NIC left at the paper's 400 Gb/s RoCE for comparability.
B200 = {"name": "B200", "peak_flops": 2.25e15, "mem_bytes": PF.B200_MEM_BYTES, "mem_bw": 8.0e12,
        "nic_bw": 400e9, "price_per_hour": 8.0, "power_w": 1000,
        "price_note": "estimate (no public list price); replace before cost planning"}
MODELS = [
    {"name": "llama-2-7b", "n_params": 6738415616, "hidden_dim": 4096, "layers": 32,
     "gqa_group": 1, "bytes_per_elem": 2, "weight_bytes": 13.5e9, "num_heads": 32},
    {"name": "llama-2-70b", "n_params": 68976648192, "hidden_dim": 8192, "layers": 80,
     "gqa_group": 8, "bytes_per_elem": 2, "weight_bytes": 138e9, "num_heads": 64},
]
SPECS = {"llama-2-7b": PF.LLAMA2_7B, "llama-2-70b": PF.LLAMA2_70B}


def last_json(path: str) -> dict:
    return json.loads([ln for ln in open(path) if ln.startswith("{")][-1])


def measured(path: str) -> dict:
    r = last_json(path)
    kv_gbs = r["value"] / r["n_gpus"]          # per GPU
    return {"source": path, "workload": r["config"]["workload"],
            "attn_mbu": round(kv_gbs * 1e9 / B200["mem_bw"], 4),
            "attn_kv_gbs_per_gpu": kv_gbs,
            "ta_ms_per_layer": r["ms_per_step"] / r["config"]["layers"],
            "e2e_kv_gbs_per_gpu": r.get("e2e", {}).get("value", 0.0) / r["n_gpus"]}


def main(c3: str, c2: str, net: str) -> None:
    m70, m7 = measured(c3), measured(c2)
    preset = last_json(net)
    cap = []
    for name, spec in SPECS.items():
        for gpus in (1, 2, 4, 8):
            for l in (4096, 32768):
                cap.append({"model": name, "gpus": gpus, "seq_len": l,
                            "max_batch": PF.max_batch(gpus * B200["mem_bytes"], 0.0, spec, l)})
    out = {
        "devices": [B200],
        "models": MODELS,
        "net_presets": [{k: preset[k] for k in ("name", "base_latency_s", "achievable_bw")}
                        | {"how": preset.get("how", "")},
                        {"name": "FHBN", "base_latency_s": 16.5e-6, "achievable_bw": 45.7e9,
                         "how": "reference net.cpp:13-18 (400 Gb/s RoCE ping-pong)"},
                        {"name": "NCCL-GDR", "base_latency_s": 33.3e-6, "achievable_bw": 35.5e9,
                         "how": "reference net.cpp:13-18"}],
        "measured": {"llama-2-70b": m70, "llama-2-7b": m7,
                     "usage": "DISAGG_CATALOG=<this file> disagg <cmd> --attn-mbu <attn_mbu> (or --ta-ms "
                              "<ta_ms_per_layer> x layers); NVLINK-PEER needs the one-line preset of "
                              "INTEGRATION.md §4 in net.cpp"},
        "capacity": {"rule": "max_batch(pool = gpus x mem_bytes, weights = 0 (a memory-pool GPU holds "
                             "no weights), headroom 0.05) — perf.cpp:130-140", "points": cap},
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(*(sys.argv[1:4] if len(sys.argv) > 3 else
           ("profiles/r02/bench_c3_n1.json", "profiles/r02/bench_c2_n1.json",
            "profiles/r02/nvlink_preset.json")))
