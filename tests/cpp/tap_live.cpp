// Live boundary test (CPU, needs /root/reference): runs the UNMODIFIED
// reference engine with EspTapPolicy wrapped around the reference's own
// policy, driving a placement-only B200 runtime through the C-ABI. The tap
// verifies page tables against Request.placement at every schedule() call;
// afterwards the event log must equal an untapped run's event-by-event
// (events.hpp:49 operator==).
#include <cstdio>
#include <iostream>
#include <set>

#include "espsim/config.hpp"
#include "espsim/cost_model.hpp"
#include "espsim/engine.hpp"
#include "espsim/trace.hpp"
#include "esp_tap_policy.hpp"

using namespace espsim;

int run(const char* policy, int instances, TokenCount cap, std::vector<TraceRecord> trace,
        const std::string& sib_path) {
  EngineParams params;
  params.exact_output_reservation = true;
  ModelConfig model;
  Engine plain(KvPool(instances, cap), model, Sib::load(sib_path),
               make_policy(parse_policy(policy)), params);
  plain.submit(trace);
  plain.run();

  esp_model_config cfg{32, 4096, 32, 128, 11008, 32000, 1e-5f, 10000.f, 1234};
  esp_runtime* rt = nullptr;
  if (esp_runtime_create(&cfg, instances, nullptr, cap, &rt) != ESP_OK) {
    std::cerr << "create: " << esp_last_error() << "\n";
    return 2;
  }
  auto tap = std::make_unique<esp_integration::EspTapPolicy>(make_policy(parse_policy(policy)),
                                                             rt, false);
  auto* tp = tap.get();
  Engine tapped(KvPool(instances, cap), model, Sib::load(sib_path), std::move(tap), params);
  tapped.submit(trace);
  tapped.run();
  const auto& a = plain.log().events();
  const auto& b = tapped.log().events();
  if (a.size() != b.size()) {
    std::cerr << "event count differs\n";
    return 1;
  }
  for (size_t i = 0; i < a.size(); ++i) {
    if (!(a[i] == b[i])) {
      std::cerr << "event " << i << " differs\n";
      return 1;
    }
  }
  // After the last decision the tap's reconcile has not run: do it via the
  // final state (every request finished -> all slots released).
  for (const auto& r : tapped.state().requests) esp_free_request(rt, r.id);
  for (int i = 0; i < instances; ++i) {
    int64_t c = 0, u = 0;
    esp_instance_info(rt, i, &c, &u);
    if (u != 0) {
      std::cerr << "instance " << i << " leaks " << u << " slots\n";
      return 1;
    }
  }
  std::printf("%s: %zu events identical, %lld decisions, %lld page-table checks, "
              "%lld prefills in fill order, %lld reconcile queries\n", policy,
              a.size(), static_cast<long long>(tp->decisions()),
              static_cast<long long>(tp->verified_requests()),
              static_cast<long long>(tp->fill_ordered_prefills()),
              static_cast<long long>(tp->reconcile_queries()));
  esp_runtime_destroy(rt);
  return 0;
}

// usage: tap_live <reference root> [sib.jsonl]   (default: the reference's default SIB)
int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: tap_live <reference root> [sib.jsonl]\n");
    return 2;
  }
  const std::string sib =
      argc > 2 ? std::string(argv[2]) : std::string(argv[1]) + "/proj/configs/default_sib.jsonl";
  int rc = run("esp", 2, 200000, {{0, 4096, 64}}, sib);
  TraceSpec spec;
  spec.distribution = "mixed";
  spec.requests_per_s = 1.0;
  spec.count = 300;
  spec.seed = 7;
  rc |= run("esp", 8, 317000, gen_trace(spec), sib);
  rc |= run("static-hybrid:2", 8, 300000, {{0, 32768, 4}, {5, 1000, 3}}, sib);
  // Tight pools: finishes, evictions and displaced-KV moves between two
  // schedule() calls (the tap frees before it moves).
  spec.requests_per_s = 4.0;
  spec.count = 120;
  spec.seed = 3;
  rc |= run("esp", 4, 60000, gen_trace(spec), sib);
  // SURVEY §8 f3 baselines on the same data path: chunked prefill (chunks
  // ride on decode steps) and disaggregation (engine-internal handoff moves).
  spec.requests_per_s = 2.0;
  spec.count = 60;
  spec.seed = 11;
  rc |= run("chunked:2048", 8, 317000, gen_trace(spec), sib);
  rc |= run("disagg:2+6", 8, 317000, gen_trace(spec), sib);
  return rc;
}
