// Live drop-in run on the GPU box: the UNMODIFIED reference engine and ESP
// scheduler (compiled here from /root/reference by oracle/Makefile into
// oracle/_ref/, a build artefact that travels with the repo snapshot) drive a
// DEVICE runtime through EspTapPolicy — every PrefillPlan, DecodeStepPlan and
// KvMove executes real sm_100a kernels on the tiny Llama shape (the
// LWM-7B KV of these traces needs 8 GPUs). The tap checks the device page
// tables against Request.placement at every schedule() call; afterwards the
// event log must equal an untapped run's event-by-event (events.hpp:49
// operator==) and the device slot recount must agree with the host counters.
//
// usage: tap_gpu <default_sib.jsonl>
#include <chrono>
#include <cstdio>
#include <iostream>

#include "espsim/config.hpp"
#include "espsim/cost_model.hpp"
#include "espsim/engine.hpp"
#include "espsim/trace.hpp"
#include "esp_tap_policy.hpp"

using namespace espsim;

namespace {

int run(const char* name, const char* policy, int instances, TokenCount cap, bool exact_output,
        std::vector<TraceRecord> trace, const std::string& sib_path, int tp_degree = 1) {
  EngineParams params;
  params.exact_output_reservation = exact_output;
  params.bandwidth_tokens_per_ms = 800;
  ModelConfig model;  // the engine accounts KV in LWM-7B bytes (cluster.hpp:29-34)
  Engine plain(KvPool(instances, cap), model, Sib::load(sib_path),
               make_policy(parse_policy(policy)), params);
  plain.submit(trace);
  plain.run();

  // Tiny Llama (2 layers, d=512, 8 x 64 heads, FFN 1536, V=32000).
  esp_model_config cfg{2, 512, 8, 64, 1536, 32000, 1e-5f, 10000.f, 1234};
  std::vector<int32_t> devices(static_cast<size_t>(instances), 0);
  esp_runtime* rt = nullptr;
  // tp > 1: tensor-parallel instances (every instance spans tp planes, here
  // all on GPU 0) — the engine and the tap are unchanged.
  std::vector<int32_t> planes(static_cast<size_t>(tp_degree), 0);
  const int made = tp_degree > 1
                       ? esp_runtime_create_tp(&cfg, instances, tp_degree, planes.data(), cap, &rt)
                          : esp_runtime_create(&cfg, instances, devices.data(), cap, &rt);
  if (made != ESP_OK) {
    std::cerr << "create: " << esp_last_error() << "\n";
    return 2;
  }
  auto tap = std::make_unique<esp_integration::EspTapPolicy>(make_policy(parse_policy(policy)),
                                                             rt, /*with_tokens=*/true);
  auto* tp = tap.get();
  Engine tapped(KvPool(instances, cap), model, Sib::load(sib_path), std::move(tap), params);
  tapped.submit(trace);
  const auto t0 = std::chrono::steady_clock::now();
  tapped.run();
  const double wall_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const auto& a = plain.log().events();
  const auto& b = tapped.log().events();
  if (a.size() != b.size()) {
    std::cerr << name << ": event count differs (" << a.size() << " vs " << b.size() << ")\n";
    return 1;
  }
  for (size_t i = 0; i < a.size(); ++i) {
    if (!(a[i] == b[i])) {
      std::cerr << name << ": event " << i << " differs\n";
      return 1;
    }
  }
  if (esp_check_conservation(rt) != ESP_OK) {
    std::cerr << name << ": conservation: " << esp_last_error() << "\n";
    return 1;
  }
  int64_t prompt = 0, gen = 0;
  for (const auto& r : tapped.state().requests) {
    if (r.phase == Phase::kFinished) {
      prompt += r.input_len;
      gen += r.generated;
    }
  }
  for (const auto& r : tapped.state().requests) esp_free_request(rt, r.id);
  for (int i = 0; i < instances; ++i) {
    int64_t c = 0, u = 0;
    esp_instance_info(rt, i, &c, &u);
    if (u != 0) {
      std::cerr << name << ": instance " << i << " leaks " << u << " slots\n";
      return 1;
    }
  }
  std::printf(
      "%s: %zu events identical, %lld decisions executed on the GPU, %lld page-table checks, "
      "%lld prompt + %lld generated tokens, %.2f s wall\n",
      name, a.size(), static_cast<long long>(tp->decisions()),
      static_cast<long long>(tp->verified_requests()), static_cast<long long>(prompt),
      static_cast<long long>(gen), wall_s);
  esp_runtime_destroy(rt);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: tap_gpu <default_sib.jsonl>\n";
    return 2;
  }
  const std::string sib = argv[1];
  // BASELINE config 1: 4K-token prompt, 2 instances, 64 decode steps.
  int rc = run("config1", "esp", 2, 200000, true, {{0, 4096, 64}}, sib);
  // Same prompt on 2 x 4096 slots: scale-down 2->1, then scale-up 1->2 mid-decode.
  rc |= run("config1_tight", "esp", 2, 4096, true, {{0, 4096, 64}}, sib);
  // BASELINE config 5: mixed trace, 8 instances x 317,000 slots.
  TraceSpec spec;
  spec.distribution = "mixed";
  spec.requests_per_s = 0.5;
  spec.count = 24;
  spec.seed = 7;
  rc |= run("config5_mixed", "esp", 8, 317000, false, gen_trace(spec), sib);
  // A denser mixed trace (96 requests at 2 req/s) on tighter instances: more
  // concurrent groups, multi-request ring batches, masters rotating.
  spec.requests_per_s = 2.0;
  spec.count = 96;
  spec.seed = 11;
  rc |= run("mixed_96", "esp", 8, 160000, true, gen_trace(spec), sib);
  // SURVEY §8 f3 baselines on the same kernels: chunked prefill (2048-token
  // chunks ride on decode steps of one 8-instance group) and prefill/decode
  // disaggregation (2 prefill + 6 decode instances, handoff KV moves).
  spec.requests_per_s = 1.0;
  spec.count = 48;
  spec.seed = 5;
  rc |= run("chunked_48", "chunked:2048", 8, 160000, true, gen_trace(spec), sib);
  rc |= run("disagg_48", "disagg:2+6", 8, 160000, true, gen_trace(spec), sib);
  // the same engine and tap over tensor-parallel instances
  // (tp = 2 planes): config 1, the config-5 mixed trace, chunked prefill
  // (chunks on tp decode steps), disaggregation with its handoff KV moves.
  rc |= run("config1_tp2", "esp", 2, 200000, true, {{0, 4096, 64}}, sib, 2);
  spec.requests_per_s = 0.5;
  spec.count = 24;
  spec.seed = 7;
  rc |= run("config5_mixed_tp2", "esp", 8, 317000, false, gen_trace(spec), sib, 2);
  spec.requests_per_s = 1.0;
  spec.count = 48;
  spec.seed = 5;
  rc |= run("chunked_48_tp2", "chunked:2048", 8, 160000, true, gen_trace(spec), sib, 2);
  rc |= run("disagg_48_tp2", "disagg:2+6", 8, 160000, true, gen_trace(spec), sib, 2);
  return rc;
}
