// Control-plane timing (SURVEY §8 d, "CPU path timing (i)"): the reference
// engine + ESP scheduler (espsim_core, single-threaded by design,
// engine.hpp:45) on a 2000-request mixed trace, timed with steady_clock,
//   untapped : the reference alone (a counting decorator counts schedule() calls)
//   tapped   : EspTapPolicy over a placement-only runtime — the drop-in's host
//              cost per iteration (reconcile, page-table verification of every
//              live request, executing each decision's page-table effects),
//              and again with verification off (set_verify_every(0))
// Prints one JSON object. Built by oracle/Makefile into oracle/_ref/.
// usage: control_plane_bench <default_sib.jsonl> [requests]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>

#include "espsim/config.hpp"
#include "espsim/cost_model.hpp"
#include "espsim/engine.hpp"
#include "espsim/trace.hpp"
#include "esp_tap_policy.hpp"

using namespace espsim;

namespace {

class Counting final : public Policy {
 public:
  explicit Counting(std::unique_ptr<Policy> inner) : inner_(std::move(inner)) {}
  std::string name() const override { return inner_->name(); }
  void init(SimState& s, const Sib& sib, const SchedulerParams& p) override {
    Policy::init(s, sib, p);
    inner_->init(s, sib, p);
  }
  std::optional<std::string> admit(const SimState& s, const Request& r) const override {
    return inner_->admit(s, r);
  }
  ScheduleDecision schedule(const SimState& s, const BandwidthModel& bw) override {
    ++calls;
    return inner_->schedule(s, bw);
  }
  int64_t calls = 0;

 private:
  std::unique_ptr<Policy> inner_;
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: control_plane_bench <default_sib.jsonl> [requests]\n";
    return 2;
  }
  const std::string sib_path = argv[1];
  TraceSpec spec;
  spec.distribution = "mixed";
  spec.requests_per_s = 1.0;
  spec.count = argc > 2 ? std::atoi(argv[2]) : 2000;
  spec.seed = 7;
  const auto trace = gen_trace(spec);
  const int instances = 8;
  const TokenCount cap = 317000;
  EngineParams params;
  params.bandwidth_tokens_per_ms = 800;
  ModelConfig model;

  auto counting = std::make_unique<Counting>(make_policy(parse_policy("esp")));
  Counting* cp = counting.get();
  Engine plain(KvPool(instances, cap), model, Sib::load(sib_path), std::move(counting), params);
  plain.submit(trace);
  auto t0 = std::chrono::steady_clock::now();
  plain.run();
  const double t_plain = seconds_since(t0);

  esp_model_config cfg{32, 4096, 32, 128, 11008, 32000, 1e-5f, 10000.f, 1234};
  esp_runtime* rt = nullptr;
  if (esp_runtime_create(&cfg, instances, nullptr, cap, &rt) != ESP_OK) {
    std::cerr << "create: " << esp_last_error() << "\n";
    return 2;
  }
  auto tap = std::make_unique<esp_integration::EspTapPolicy>(make_policy(parse_policy("esp")), rt,
                                                             /*with_tokens=*/false);
  auto* tp = tap.get();
  Engine tapped(KvPool(instances, cap), model, Sib::load(sib_path), std::move(tap), params);
  tapped.submit(trace);
  t0 = std::chrono::steady_clock::now();
  tapped.run();
  const double t_tap = seconds_since(t0);
  const bool same = plain.log().events() == tapped.log().events();
  esp_runtime_destroy(rt);

  // The same with page-table verification off: the tap's execution cost alone.
  esp_runtime* rt2 = nullptr;
  if (esp_runtime_create(&cfg, instances, nullptr, cap, &rt2) != ESP_OK) {
    std::cerr << "create: " << esp_last_error() << "\n";
    return 2;
  }
  auto tap2 = std::make_unique<esp_integration::EspTapPolicy>(make_policy(parse_policy("esp")),
                                                              rt2, /*with_tokens=*/false);
  tap2->set_verify_every(0);
  Engine tapped2(KvPool(instances, cap), model, Sib::load(sib_path), std::move(tap2), params);
  tapped2.submit(trace);
  t0 = std::chrono::steady_clock::now();
  tapped2.run();
  const double t_tap2 = seconds_since(t0);
  const bool same2 = plain.log().events() == tapped2.log().events();
  esp_runtime_destroy(rt2);
  const double it = static_cast<double>(cp->calls);
  std::printf(
      "{\"trace\": \"mixed, %lld requests at 1 req/s, seed 7, 8 instances x %lld slots, esp\", "
      "\"iterations\": %lld, \"events\": %zu, \"events_identical\": %s, "
      "\"untapped_ms\": %.3f, \"untapped_us_per_iteration\": %.3f, "
      "\"tapped_ms\": %.3f, \"tapped_us_per_iteration\": %.3f, "
      "\"tap_overhead_us_per_iteration\": %.3f, \"page_table_checks\": %lld, "
      "\"tapped_no_verify_ms\": %.3f, \"tap_overhead_no_verify_us_per_iteration\": %.3f, "
      "\"threads\": 1}\n",
      static_cast<long long>(spec.count), static_cast<long long>(cap),
      static_cast<long long>(cp->calls), plain.log().events().size(), same ? "true" : "false",
      t_plain * 1e3, t_plain * 1e6 / it, t_tap * 1e3, t_tap * 1e6 / it,
      (t_tap - t_plain) * 1e6 / it, static_cast<long long>(tp->verified_requests()),
      t_tap2 * 1e3, (t_tap2 - t_plain) * 1e6 / it);
  return same && same2 ? 0 : 1;
}
