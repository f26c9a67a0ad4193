// EspTapPolicy — the drop-in boundary on the reference side.
//
// A decorator over the reference's only plugin interface, espsim::Policy
// (proj/include/espsim/policies.hpp:43-71), injected through Engine's
// constructor (engine.hpp:48-49). Engine::run calls policy_->schedule() and
// immediately apply_decision() with nothing in between (engine.cpp:680-681),
// so a decision seen here is exactly the decision the engine commits. For
// every decision the tap drives the B200 runtime through the C-ABI
// (include/esp_abi.h) in apply_decision's order (engine.cpp:246-490):
//   MigrationPlan.moves -> esp_move_kv         (engine.cpp:260-309)
//   PrefillPlan         -> esp_prefill          (engine.cpp:311-363)
//   DecodeStepPlan      -> esp_decode_step      (engine.cpp:365-489)
// and before that reconciles the changes the engine makes outside
// apply_decision: finished / rejected / evicted requests are freed
// (engine.cpp:119-166) and "displaced" KV (resolve_foreign_kv,
// engine.cpp:587-648) is moved. It then verifies that every request's device
// page table equals Request.placement and every instance's used slots equal
// ElasticInstance.kv_used, throwing espsim::InternalError on any mismatch —
// the engine aborts exactly as on its own conservation failure
// (cluster.cpp:113-132). Decisions are returned unchanged, so the engine's
// behaviour (and its event log) is identical to the untapped run.
//
// Header-only; include after the espsim headers and link libesp_b200.so.
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "esp_abi.h"
#include "espsim/policies.hpp"
#include "espsim/state.hpp"

namespace esp_integration {

// Prompt token ids of a request (the simulator's requests carry none).
using TokenSource = std::function<std::vector<int32_t>(espsim::RequestId, espsim::TokenCount)>;

inline std::vector<int32_t> synthetic_tokens(espsim::RequestId id, espsim::TokenCount n,
                                             int32_t vocab = 32000) {
  std::mt19937_64 rng(0x5eedULL ^ static_cast<uint64_t>(id));
  std::vector<int32_t> t(static_cast<size_t>(n));
  for (auto& x : t) x = static_cast<int32_t>(rng() % static_cast<uint64_t>(vocab));
  return t;
}

// Maps a C-ABI status onto the reference's exception taxonomy.
inline void check(int rc) {
  if (rc == ESP_OK) return;
  const std::string msg = std::string("esp: ") + esp_last_error();
  switch (rc) {
    case ESP_ERR_CONFIG: throw espsim::ConfigError(msg);
    case ESP_ERR_INFEASIBLE: throw espsim::InfeasiblePlanError(msg);
    case ESP_ERR_UNKNOWN_STRATEGY: throw espsim::UnknownStrategyError(msg);
    default: throw espsim::InternalError(msg);
  }
}

class EspTapPolicy final : public espsim::Policy {
 public:
  EspTapPolicy(std::unique_ptr<espsim::Policy> inner, esp_runtime* rt, bool with_tokens,
               TokenSource tokens = nullptr)
      : inner_(std::move(inner)), rt_(rt), with_tokens_(with_tokens),
        tokens_(tokens ? std::move(tokens) : TokenSource([](espsim::RequestId r, espsim::TokenCount n) {
          return synthetic_tokens(r, n);
        })) {}

  std::string name() const override { return inner_->name(); }

  void init(espsim::SimState& state, const espsim::Sib& sib,
            const espsim::SchedulerParams& params) override {
    Policy::init(state, sib, params);
    inner_->init(state, sib, params);
  }

  std::optional<std::string> admit(const espsim::SimState& state,
                                   const espsim::Request& req) const override {
    return inner_->admit(state, req);
  }

  espsim::ScheduleDecision schedule(const espsim::SimState& state,
                                    const espsim::BandwidthModel& bw) override {
    reconcile(state);
    if (verify_every_ > 0 && calls_++ % verify_every_ == 0) verify(state);
    espsim::ScheduleDecision d = inner_->schedule(state, bw);
    execute(state, d);
    ++decisions_;
    return d;
  }

  // Page-table verification on every n-th schedule() call (1, the default:
  // every call; 0: never — the tap then only reconciles and executes).
  void set_verify_every(int64_t n) { verify_every_ = n; }
  int64_t decisions() const { return decisions_; }
  // Requests whose device page table reconcile() had to query (the engine's
  // placement differed from what the tap's own operations predict).
  int64_t reconcile_queries() const { return queried_; }
  int64_t verified_requests() const { return verified_; }
  // Prefill plans passed in the restated fill order (vs map order).
  int64_t fill_ordered_prefills() const { return fill_ordered_; }

 private:
  std::map<int32_t, int64_t> device_placement(espsim::RequestId r) const {
    // esp_query_placement reports the full count; grow the buffer and ask
    // again when a request spans more instances than it holds.
    int32_t n = 0;
    check(esp_query_placement(rt_, r, pl_inst_.data(), pl_tok_.data(),
                              static_cast<int32_t>(pl_inst_.size()), &n));
    if (n > static_cast<int32_t>(pl_inst_.size())) {
      pl_inst_.resize(static_cast<size_t>(n));
      pl_tok_.resize(static_cast<size_t>(n));
      check(esp_query_placement(rt_, r, pl_inst_.data(), pl_tok_.data(), n, &n));
    }
    std::map<int32_t, int64_t> m;
    for (int32_t i = 0; i < n; ++i) m[pl_inst_[static_cast<size_t>(i)]] = pl_tok_[static_cast<size_t>(i)];
    return m;
  }

  void reconcile(const espsim::SimState& s) {
    // Pass 1: release every finished / rejected / evicted request first, so
    // the displaced-KV moves of pass 2 can land in the slots they freed (the
    // engine frees before it displaces, engine.cpp:119-166 / :587-648).
    for (auto it = live_.begin(); it != live_.end();) {
      const espsim::Request& q = s.requests[static_cast<size_t>(*it)];
      if (q.phase == espsim::Phase::kFinished || q.phase == espsim::Phase::kRejected ||
          q.placement.empty()) {
        check(esp_free_request(rt_, *it));  // finish / evict-and-recompute
        known_.erase(*it);
        it = live_.erase(it);
      } else {
        ++it;
      }
    }
    // Pass 2: engine-internal KV moves (displaced KV): surplus -> deficit.
    // known_ mirrors what the tap itself did to the device (prefill
    // placements, appends at the master assign_masters picks, moves); a
    // request whose engine placement equals it needs no device query. Any
    // other difference (an engine-internal move, or a mirror that is off) is
    // resolved against the device's own page table, so the mirror is only a
    // shortcut, never the source of truth.
    for (espsim::RequestId r : live_) {
      const espsim::Request& q = s.requests[static_cast<size_t>(r)];
      auto kn = known_.find(r);
      if (kn != known_.end() && same_placement(kn->second, q.placement)) continue;
      auto have = device_placement(r);
      std::vector<std::pair<int32_t, int64_t>> surplus, deficit;
      std::set<int32_t> ids;
      for (auto& kv : have) ids.insert(kv.first);
      for (auto& kv : q.placement) ids.insert(kv.first);
      for (int32_t i : ids) {
        const int64_t h = have.count(i) ? have[i] : 0;
        const int64_t w = q.placement.count(i) ? q.placement.at(i) : 0;
        if (h > w) surplus.emplace_back(i, h - w);
        if (w > h) deficit.emplace_back(i, w - h);
      }
      size_t a = 0, b = 0;
      while (a < surplus.size() && b < deficit.size()) {
        const int64_t mv = std::min(surplus[a].second, deficit[b].second);
        check(esp_move_kv(rt_, r, surplus[a].first, deficit[b].first, mv));
        if ((surplus[a].second -= mv) == 0) ++a;
        if ((deficit[b].second -= mv) == 0) ++b;
      }
      known_[r] = std::map<int32_t, int64_t>(q.placement.begin(), q.placement.end());
      ++queried_;
    }
  }

  template <class P>
  static bool same_placement(const std::map<int32_t, int64_t>& a, const P& b) {
    if (a.size() != b.size()) return false;
    auto i = a.begin();
    for (const auto& kv : b) {
      if (i->first != kv.first || i->second != kv.second) return false;
      ++i;
    }
    return true;
  }
  static void add_tokens(std::map<int32_t, int64_t>& m, int32_t inst, int64_t n) {
    if ((m[inst] += n) == 0) m.erase(inst);
  }

  // The plan's placement pairs in TOKEN (fill) order: plan_prefill_scale_down
  // (scheduler.cpp:663-713) lays each request's tokens contiguously over the
  // survivors ordered by (free desc, id asc), one cursor across the batch.
  // The PrefillPlan only keeps per-instance counts (a KvPlacement map), so
  // the order is recomputed with the planner's restatement over the
  // runtime's free slots (the scheduler's free_after view: migrations are
  // already applied and DP batches own disjoint instances). Plans that
  // another policy laid out differently keep their map order.
  std::vector<std::vector<std::pair<int32_t, int64_t>>> fill_order(const espsim::SimState& s,
                                                                   const espsim::PrefillPlan& p) {
    const size_t n = p.requests.size(), d = p.instances.size();
    std::vector<std::vector<std::pair<int32_t, int64_t>>> out(n);
    for (size_t r = 0; r < n; ++r) {
      for (const auto& kv : p.placement.at(p.requests[r])) out[r].push_back(kv);
    }
    std::vector<int32_t> inst(p.instances.begin(), p.instances.end());
    std::vector<int64_t> free(d), lens(n);
    for (size_t i = 0; i < d; ++i) {
      int64_t cap = 0, used = 0;
      check(esp_instance_info(rt_, inst[i], &cap, &used));
      free[i] = cap - used;
    }
    for (size_t r = 0; r < n; ++r) lens[r] = s.requests[static_cast<size_t>(p.requests[r])].input_len;
    std::vector<int32_t> dec(d), pi(n * d), pn(n);
    std::vector<int64_t> pt(n * d);
    int32_t nd = 0;
    int64_t vol = 0;
    if (esp_plan_prefill_scale_down(inst.data(), free.data(), static_cast<int32_t>(d), lens.data(),
                                    static_cast<int32_t>(n), dec.data(), &nd, pi.data(), pt.data(),
                                    pn.data(), &vol) != ESP_OK) {
      return out;
    }
    std::vector<std::vector<std::pair<int32_t, int64_t>>> fill(n);
    for (size_t r = 0; r < n; ++r) {
      std::map<int32_t, int64_t> counts;
      for (int32_t j = 0; j < pn[r]; ++j) {
        fill[r].emplace_back(pi[r * d + j], pt[r * d + j]);
        counts[pi[r * d + j]] += pt[r * d + j];
      }
      const auto& want = p.placement.at(p.requests[r]);
      if (!std::equal(counts.begin(), counts.end(), want.begin(), want.end(),
                      [](const auto& x, const auto& y) { return x.first == y.first && x.second == y.second; }) ||
          counts.size() != want.size()) {
        return out;
      }
    }
    ++fill_ordered_;
    return fill;
  }

  void verify(const espsim::SimState& s) {
    for (espsim::RequestId r : live_) {
      std::map<int32_t, int64_t> want(s.requests[static_cast<size_t>(r)].placement.begin(),
                                      s.requests[static_cast<size_t>(r)].placement.end());
      if (device_placement(r) != want) {
        throw espsim::InternalError("device page table of request " + std::to_string(r) +
                                    " drifted from its KV placement");
      }
      ++verified_;
    }
    for (const auto& inst : s.pool.instances()) {
      int64_t cap = 0, used = 0;
      check(esp_instance_info(rt_, inst.id, &cap, &used));
      if (used != inst.kv_used) {
        throw espsim::InternalError("device slots of instance " + std::to_string(inst.id) +
                                    " drifted from kv_used");
      }
    }
  }

  void execute(const espsim::SimState& s, const espsim::ScheduleDecision& d) {
    for (const espsim::MigrationPlan& m : d.migrations) {
      for (const espsim::KvMove& mv : m.moves) {
        check(esp_move_kv(rt_, mv.request, mv.from, mv.to, mv.tokens));
        auto kn = known_.find(mv.request);
        if (kn != known_.end()) {
          add_tokens(kn->second, mv.from, -mv.tokens);
          add_tokens(kn->second, mv.to, mv.tokens);
        }
      }
    }
    for (const espsim::PrefillPlan& p : d.prefills) {
      std::vector<int64_t> ids(p.requests.begin(), p.requests.end()), lens;
      std::vector<int32_t> ring(p.instances.begin(), p.instances.end()), rn, ri, toks;
      std::vector<int64_t> rt;
      const auto order = fill_order(s, p);
      for (size_t k = 0; k < p.requests.size(); ++k) {
        const espsim::RequestId r = p.requests[k];
        const espsim::TokenCount n = s.requests[static_cast<size_t>(r)].input_len;
        lens.push_back(n);
        rn.push_back(static_cast<int32_t>(order[k].size()));
        auto& kn = known_[r];
        kn.clear();
        for (const auto& [inst, tok] : order[k]) {
          ri.push_back(inst);
          rt.push_back(tok);
          add_tokens(kn, inst, tok);
        }
        if (with_tokens_) {
          auto t = tokens_(r, n);
          toks.insert(toks.end(), t.begin(), t.end());
        }
        live_.insert(r);
      }
      esp_prefill_args a{};
      a.n_requests = static_cast<int32_t>(ids.size());
      a.request_ids = ids.data();
      a.input_lens = lens.data();
      a.tokens = with_tokens_ ? toks.data() : nullptr;
      a.dop = static_cast<int32_t>(ring.size());
      a.ring = ring.data();
      a.retain_n = rn.data();
      a.retain_instance = ri.data();
      a.retain_tokens = rt.data();
      check(esp_prefill(rt_, &a));
    }
    for (const espsim::DecodeStepPlan& p : d.decode_steps) {
      const espsim::GroupState& gs = s.groups.at(p.group);
      std::vector<int32_t> members(gs.group.instances.begin(), gs.group.instances.end());
      members.insert(members.end(), p.add_instances.begin(), p.add_instances.end());
      std::sort(members.begin(), members.end());
      std::vector<int32_t> masters(p.masters.begin(), p.masters.end());
      std::vector<int64_t> batch(gs.batch.begin(), gs.batch.end());
      const bool chunk = p.chunk_request >= 0 && p.chunk_tokens > 0;
      if (batch.empty() && !chunk) continue;
      esp_decode_args a{};
      a.n_members = static_cast<int32_t>(members.size());
      a.members = members.data();
      a.n_masters = static_cast<int32_t>(masters.size());
      a.masters = masters.data();
      a.batch_size = static_cast<int32_t>(batch.size());
      a.batch = batch.data();
      // Chunked prefill riding on the step (engine.cpp:432-462, 570-579).
      std::vector<int32_t> ci, ctoks;
      std::vector<int64_t> ct;
      if (chunk) {
        const espsim::Request& q = s.requests[static_cast<size_t>(p.chunk_request)];
        for (const auto& [inst, tok] : p.chunk_placement) {
          ci.push_back(inst);
          ct.push_back(tok);
        }
        auto& kn = known_[p.chunk_request];
        for (const auto& [inst, tok] : p.chunk_placement) add_tokens(kn, inst, tok);
        a.chunk_request = p.chunk_request;
        a.chunk_tokens = p.chunk_tokens;
        a.chunk_n = static_cast<int32_t>(ci.size());
        a.chunk_instance = ci.data();
        a.chunk_tokens_on = ct.data();
        a.chunk_final = q.prefilled + p.chunk_tokens == q.input_len ? 1 : 0;
        if (with_tokens_) {
          const auto all = tokens_(p.chunk_request, q.input_len);
          ctoks.assign(all.begin() + q.prefilled, all.begin() + q.prefilled + p.chunk_tokens);
          a.chunk_token_ids = ctoks.data();
        }
        live_.insert(p.chunk_request);
      }
      check(esp_decode_step(rt_, &a));
      // the step appended one token per batch request at its master
      // (assign_masters, esp_mechanics.cpp:220-238, as the runtime does)
      if (!batch.empty()) {
        std::vector<int32_t> master_of(batch.size());
        check(esp_assign_masters(batch.data(), static_cast<int32_t>(batch.size()), masters.data(),
                                 static_cast<int32_t>(masters.size()), master_of.data()));
        for (size_t i = 0; i < batch.size(); ++i) {
          auto kn = known_.find(batch[i]);
          if (kn != known_.end()) add_tokens(kn->second, master_of[i], 1);
        }
      }
    }
  }

  std::unique_ptr<espsim::Policy> inner_;
  esp_runtime* rt_;
  bool with_tokens_;
  TokenSource tokens_;
  std::set<espsim::RequestId> live_;
  std::map<espsim::RequestId, std::map<int32_t, int64_t>> known_;
  int64_t queried_ = 0;
  int64_t decisions_ = 0;
  int64_t verified_ = 0;
  int64_t fill_ordered_ = 0;
  mutable std::vector<int32_t> pl_inst_ = std::vector<int32_t>(16);
  mutable std::vector<int64_t> pl_tok_ = std::vector<int64_t>(16);
  int64_t verify_every_ = 1;
  int64_t calls_ = 0;
};

}  // namespace esp_integration
