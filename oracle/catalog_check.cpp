// oracle/catalog_check.cpp — TEST INFRASTRUCTURE (planner feedback, §8(f) rows 3-4).
//
// Loads integration/b200_catalog.json through the reference's OWN loaders and validators
// (load_device_spec / load_llm_spec, core/src/model.cpp; DeviceSpec / LlmSpec::validate) and
// evaluates the reference's own capacity planner for it (max_batch, core/src/perf.cpp:130-140;
// kv_bytes_per_token, perf.cpp:123-128), printing one JSON object per line for
// tests/test_planner_cpu.py.  Built by oracle/Makefile from the reference sources in place.
#include <cstdio>
#include <fstream>
#include <iostream>

#include "disagg/model.hpp"
#include "disagg/perf.hpp"

using disagg::json;

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s catalog.json\n", argv[0]);
    return 2;
  }
  std::ifstream f(argv[1]);
  const json doc = json::parse(f);
  for (const auto& d : doc.at("devices")) {
    const disagg::DeviceSpec dev = disagg::load_device_spec(d);  // validates
    std::printf("{\"device\": \"%s\", \"mem_bytes\": %.17g, \"mem_bw\": %.17g}\n", dev.name.c_str(),
                dev.mem_bytes, dev.mem_bw);
    for (const auto& m : doc.at("models")) {
      const disagg::LlmSpec spec = disagg::load_llm_spec(m);  // validates
      for (int gpus : {1, 2, 4, 8})
        for (long long l : {4096LL, 32768LL}) {
          const double pool = gpus * dev.mem_bytes;
          long long b = -1;
          try {
            b = disagg::max_batch(pool, 0.0, spec, l);
          } catch (const disagg::Error&) {
          }
          std::printf("{\"model\": \"%s\", \"gpus\": %d, \"seq_len\": %lld, \"kv_bytes_per_token\": "
                      "%.17g, \"max_batch\": %lld}\n",
                      spec.name.c_str(), gpus, l, disagg::kv_bytes_per_token(spec), b);
        }
    }
  }
  return 0;
}
