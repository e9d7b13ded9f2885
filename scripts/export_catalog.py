"""Export measured B200 attention numbers in the reference planner's own input formats.

The reference plans deployments analytically: attention time is
roofline_time(attn_cost, memory_pool, EfficiencyProfile, attention) (reference
core/src/sim.cpp:295-301), derated by EfficiencyProfile.attn_mbu (perf.hpp:30-35, default 0.80,
"calibration knobs, not measurements").  This script turns a bench.py result into:

  * a DISAGG_CATALOG extension file (reference tools/common.cpp:18-40) with a B200 DeviceSpec
    (model.cpp:180-193 schema) and the LLaMA-2 models BASELINE.json names (the reference
    catalog has neither, catalog.cpp:39-53);
  * the measured attention MBU to pass as --attn-mbu (main.cpp:23), and the measured per-layer
    attention time for --ta-ms (main.cpp:38, cmd_analysis.cpp:92-99).

    python scripts/export_catalog.py profiles/r01_final_bench_c3.log > integration/b200_catalog.json
"""
import json
import sys

# B200 device figures: dense bf16 peak, HBM capacity and bandwidth at spec (the planner derates
# them with the efficiency profile), NIC left at the paper's 400 Gb/s RoCE for comparability.
B200 = {"name": "B200", "peak_flops": 2.25e15, "mem_bytes": 180e9, "mem_bw": 8.0e12,
        "nic_bw": 400e9, "price_per_hour": 0.0, "power_w": 1000,
        "price_note": "price not listed; set before cost planning"}
MODELS = [
    {"name": "llama-2-7b", "n_params": 6738415616, "hidden_dim": 4096, "layers": 32,
     "gqa_group": 1, "bytes_per_elem": 2, "weight_bytes": 13.5e9, "num_heads": 32},
    {"name": "llama-2-70b", "n_params": 68976648192, "hidden_dim": 8192, "layers": 80,
     "gqa_group": 8, "bytes_per_elem": 2, "weight_bytes": 138e9, "num_heads": 64},
]


def main(path: str) -> None:
    line = next(ln for ln in open(path) if ln.startswith("{"))
    r = json.loads(line)
    kv_gbs = r["value"] / r["n_gpus"]          # per GPU
    mbu_spec = kv_gbs * 1e9 / B200["mem_bw"]    # against the DeviceSpec bandwidth
    out = {
        "devices": [B200],
        "models": MODELS,
        "measured": {
            "source": path,
            "workload": r["config"]["workload"],
            "attn_mbu": round(mbu_spec, 4),
            "attn_kv_gbs_per_gpu": kv_gbs,
            "ta_ms_per_layer": r["ms_per_step"] / r["config"]["layers"],
            "usage": "DISAGG_CATALOG=<this file> disagg <cmd> --attn-mbu <attn_mbu> "
                     "(or --ta-ms <ta_ms_per_layer> x layers for min-bandwidth)",
        },
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_final_bench_c3.log")
