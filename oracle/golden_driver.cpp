// Golden-fixture generator — TEST INFRASTRUCTURE (oracle side only).
//
// Links the UNMODIFIED reference library (compiled in place from
// /root/reference/proj/src/*.cpp by oracle/Makefile into oracle/_ref/) and
// records what the reference decides, so the B200 data path can be held to it
// on a box where /root/reference does not exist:
//
//   * mechanics_random.jsonl — seeded random inputs and the reference outputs
//     of the hot-path placement functions: plan_prefill_scale_down
//     (scheduler.cpp:663-713), plan_decode_step_core (scheduler.cpp:726-804),
//     assign_masters (esp_mechanics.cpp:220-238), decode_step_comm
//     (esp_mechanics.cpp:240-264), build_ring_schedule + coverage/volume
//     (esp_mechanics.cpp:24-70), proactive_scale_down (:78-136),
//     reactive_migrate (:138-218), kv_bytes_per_token (cluster.cpp:30-34),
//     Sib::prefill_time_sums / decode_time (cost_model.cpp:169-187).
//   * scenario_<name>.jsonl — a Policy decorator ("tap") wrapped around the
//     reference's own EspPolicy / FixedGroupsPolicy (policies.hpp:43-71,
//     injected through Engine's constructor, engine.hpp:48-49) records, at
//     every schedule() call, the engine events since the previous call, the
//     KV placement state the engine holds, and the ScheduleDecision it is
//     about to apply (engine.cpp:680-681). The replay tests drive the B200
//     runtime's C-ABI with exactly these decisions and require its page tables
//     to equal these placements at every step.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "espsim/cluster.hpp"
#include "espsim/cost_model.hpp"
#include "espsim/engine.hpp"
#include "espsim/esp_mechanics.hpp"
#include "espsim/policies.hpp"
#include "espsim/scheduler.hpp"
#include "espsim/state.hpp"
#include "espsim/trace.hpp"
#include "json.hpp"

using namespace espsim;
using json = nlohmann::json;

namespace {

json placement_json(const KvPlacement& p) {
  json a = json::array();
  for (const auto& [inst, tok] : p) a.push_back({inst, tok});
  return a;
}

const char* phase_name(Phase p) {
  switch (p) {
    case Phase::kPending: return "pending";
    case Phase::kPrefill: return "prefill";
    case Phase::kDecoding: return "decoding";
    case Phase::kFinished: return "finished";
    case Phase::kEvicted: return "evicted";
    case Phase::kRejected: return "rejected";
  }
  return "?";
}

json state_json(const SimState& s) {
  json used = json::array();
  for (const auto& inst : s.pool.instances()) used.push_back(inst.kv_used);
  json pl = json::object();
  json ph = json::object();
  for (const Request& r : s.requests) {
    ph[std::to_string(r.id)] = phase_name(r.phase);
    if (!r.placement.empty()) pl[std::to_string(r.id)] = placement_json(r.placement);
  }
  (void)ph;
  return json{{"kv_used", used}, {"placement", pl}};
}

json event_json(const Event& e) {
  return json{{"t", e.time_ms}, {"kind", event_kind_name(e.kind)},
              {"request", e.request}, {"group", e.group},
              {"tokens", e.tokens}, {"detail", e.detail}};
}

json decision_json(const ScheduleDecision& d, const SimState& s) {
  json j;
  j["rejects"] = d.rejects;
  json mig = json::array();
  for (const MigrationPlan& m : d.migrations) {
    json moves = json::array();
    for (const KvMove& mv : m.moves) moves.push_back({mv.request, mv.from, mv.to, mv.tokens});
    mig.push_back({{"group", m.group}, {"drop", m.drop}, {"volume", m.volume}, {"moves", moves}});
  }
  j["migrations"] = mig;
  json pf = json::array();
  for (const PrefillPlan& p : d.prefills) {
    json pl = json::object();
    for (const auto& [rid, place] : p.placement) pl[std::to_string(rid)] = placement_json(place);
    json lens = json::array();
    for (RequestId r : p.requests) lens.push_back(s.requests[r].input_len);
    pf.push_back({{"requests", p.requests}, {"input_lens", lens},
                  {"instances", p.instances}, {"dop", p.strategy.dop},
                  {"est_ms", p.est_ms}, {"placement", pl},
                  {"decode_instances", p.decode_instances},
                  {"decode_group", p.decode_group},
                  {"ring_volume", p.ring_volume},
                  {"reactive_handoff", p.reactive_handoff}});
  }
  j["prefills"] = pf;
  json ds = json::array();
  for (const DecodeStepPlan& p : d.decode_steps) {
    const GroupState& gs = s.groups.at(p.group);
    json step{{"group", p.group}, {"members", gs.group.instances},
              {"add_instances", p.add_instances}, {"masters", p.masters},
              {"batch", gs.batch}, {"chunk_request", p.chunk_request},
              {"chunk_tokens", p.chunk_tokens}};
    if (p.chunk_request >= 0) {
      // chunked prefill (policies.cpp:297-405): where the chunk's KV goes and
      // how much of the prompt precedes it (engine.cpp:432-462)
      const Request& q = s.requests[p.chunk_request];
      step["chunk_placement"] = placement_json(p.chunk_placement);
      step["chunk_prefilled"] = q.prefilled;
      step["chunk_input_len"] = q.input_len;
    }
    ds.push_back(step);
  }
  j["decode_steps"] = ds;
  return j;
}

// The tap: forwards to the wrapped reference policy unchanged and records.
class RecordingTap final : public Policy {
 public:
  RecordingTap(std::unique_ptr<Policy> inner, std::ostream* out)
      : inner_(std::move(inner)), out_(out) {}
  std::string name() const override { return "tap(" + inner_->name() + ")"; }
  void init(SimState& state, const Sib& sib, const SchedulerParams& params) override {
    Policy::init(state, sib, params);
    inner_->init(state, sib, params);
  }
  std::optional<std::string> admit(const SimState& state, const Request& req) const override {
    return inner_->admit(state, req);
  }
  ScheduleDecision schedule(const SimState& state, const BandwidthModel& bw) override {
    ScheduleDecision d = inner_->schedule(state, bw);
    json ev = pending_events();
    if (!d.empty() || !ev.empty()) {
      json j{{"kind", "step"}, {"k", k_}, {"clock", state.clock}, {"events", ev},
             {"before", state_json(state)}, {"decision", decision_json(d, state)}};
      *out_ << j.dump() << "\n";
      ++steps_;
    }
    ++k_;
    return d;
  }
  json pending_events() {
    json ev = json::array();
    if (!engine) return ev;
    const auto& all = engine->log().events();
    for (; seen_ < all.size(); ++seen_) ev.push_back(event_json(all[seen_]));
    return ev;
  }
  const Engine* engine = nullptr;
  int64_t steps_ = 0;

 private:
  std::unique_ptr<Policy> inner_;
  std::ostream* out_;
  int64_t k_ = 0;
  size_t seen_ = 0;
};

Sib load_default_sib(const std::string& ref) {
  return Sib::load(ref + "/proj/configs/default_sib.jsonl");
}

struct Scenario {
  std::string name;
  int instances;
  TokenCount capacity;
  ModelConfig model;
  std::string policy;
  bool exact_output = true;
  std::vector<TraceRecord> trace;
};

void run_scenario(const Scenario& sc, const std::string& ref, const std::string& outdir) {
  std::ofstream out(outdir + "/scenario_" + sc.name + ".jsonl");
  json reqs = json::array();
  for (size_t i = 0; i < sc.trace.size(); ++i) {
    reqs.push_back({{"id", i}, {"arrival_ms", sc.trace[i].arrival_ms},
                    {"input_len", sc.trace[i].input_len},
                    {"output_len", sc.trace[i].output_len}});
  }
  out << json{{"kind", "scenario"}, {"name", sc.name}, {"instances", sc.instances},
              {"kv_capacity", sc.capacity}, {"policy", sc.policy},
              {"model", {{"layers", sc.model.layers}, {"hidden_dim", sc.model.hidden_dim},
                         {"kv_heads", sc.model.kv_heads},
                         {"bytes_per_element", sc.model.bytes_per_element}}},
              {"kv_bytes_per_token", kv_bytes_per_token(sc.model)},
              {"exact_output_reservation", sc.exact_output},
              {"requests", reqs}}.dump()
      << "\n";
  EngineParams params;
  params.exact_output_reservation = sc.exact_output;
  params.bandwidth_tokens_per_ms = 800;
  auto tap = std::make_unique<RecordingTap>(make_policy(parse_policy(sc.policy)), &out);
  RecordingTap* tap_ptr = tap.get();
  Engine engine(KvPool(sc.instances, sc.capacity), sc.model, load_default_sib(ref),
                std::move(tap), params);
  tap_ptr->engine = &engine;
  engine.submit(sc.trace);
  engine.run();
  json fin{{"kind", "final"}, {"events", tap_ptr->pending_events()},
           {"state", state_json(engine.state())},
           {"n_events", engine.log().size()}};
  out << fin.dump() << "\n";
  std::cout << sc.name << ": " << tap_ptr->steps_ << " steps, " << engine.log().size()
            << " events\n";
}

// Config 4: a hand-built 4-of-8 decoding group, 16 x 65536-token requests,
// driven through esp_schedule_iteration + Engine::apply_decision for three
// steps (masters [0,1], [2,3], then scale-up 4->5).
void run_config4(const std::string& ref, const std::string& outdir) {
  const int m = 8;
  const TokenCount cap = 262152;
  std::ofstream out(outdir + "/scenario_config4_decode.jsonl");
  Sib sib = load_default_sib(ref);
  ModelConfig model;  // LWM-7B defaults (cluster.hpp:29-34)
  EngineParams params;
  params.exact_output_reservation = true;
  Engine engine(KvPool(m, cap), model, sib, make_policy(parse_policy("esp")), params);
  SimState& s = engine.mutable_state();
  GroupState gs;
  gs.group.id = 0;
  gs.group.instances = {0, 1, 2, 3};
  gs.group.masters = {0};
  json reqs = json::array();
  for (int r = 0; r < 16; ++r) {
    Request req;
    req.id = r;
    req.phase = Phase::kDecoding;
    req.input_len = 65536;
    req.output_len = 64;
    req.max_output_len = 64;
    // 16 x 65536 tokens spread evenly over the four members.
    for (int i = 0; i < 4; ++i) req.placement[i] = 16384;
    if (!s.pool.allocate(req.placement).ok) throw InternalError("config4 setup");
    req.master = 0;
    req.prefill_done_ms = 0;
    s.committed_max_tokens += req.input_len + req.max_output_len;
    s.requests.push_back(req);
    gs.batch.push_back(r);
    reqs.push_back({{"id", r}, {"arrival_ms", 0}, {"input_len", 65536}, {"output_len", 64},
                    {"placement", placement_json(req.placement)}});
  }
  for (int i = 0; i < 4; ++i) s.pool.at(i).group = 0;
  s.groups[0] = gs;
  s.next_group = 1;
  out << json{{"kind", "scenario"}, {"name", "config4_decode"}, {"instances", m},
              {"kv_capacity", cap}, {"policy", "esp"},
              {"kv_bytes_per_token", kv_bytes_per_token(model)},
              {"prebuilt", true}, {"requests", reqs}}.dump()
      << "\n";
  BandwidthModel bw(800);
  SchedulerParams sp;
  for (int step = 0; step < 3; ++step) {
    ScheduleDecision d = esp_schedule_iteration(s, sib, bw, sp);
    out << json{{"kind", "step"}, {"k", step}, {"clock", s.clock},
                {"events", json::array()}, {"before", state_json(s)},
                {"decision", decision_json(d, s)}}.dump()
        << "\n";
    engine.apply_decision(d);
    Millis t = s.clock;
    for (const auto& inst : s.pool.instances()) t = std::max(t, inst.busy_until_ms);
    s.clock = t;
  }
  json evs = json::array();
  for (const Event& e : engine.log().events()) evs.push_back(event_json(e));
  out << json{{"kind", "final"}, {"events", evs}, {"state", state_json(s)},
              {"n_events", engine.log().size()}}.dump()
      << "\n";
  std::cout << "config4_decode: 3 steps\n";
}

// ---- randomized mechanics goldens ------------------------------------------

void mechanics(const std::string& ref, const std::string& outdir) {
  std::ofstream out(outdir + "/mechanics_random.jsonl");
  std::mt19937_64 rng(20240415);
  auto rnd = [&](int64_t lo, int64_t hi) {  // inclusive
    return lo + static_cast<int64_t>(rng() % static_cast<uint64_t>(hi - lo + 1));
  };

  // plan_prefill_scale_down: random frees, random multi-request batches.
  for (int t = 0; t < 300; ++t) {
    const int m = static_cast<int>(rnd(1, 8));
    const TokenCount cap = rnd(1, 5) * 1000;
    SimState s;
    s.pool = KvPool(m, cap);
    std::vector<TokenCount> free_ov;
    std::vector<InstanceId> inst(m);
    std::iota(inst.begin(), inst.end(), 0);
    std::shuffle(inst.begin(), inst.end(), rng);
    const int d = static_cast<int>(rnd(1, m));
    inst.resize(d);
    TokenCount tot_free = 0;
    for (int i = 0; i < m; ++i) {
      TokenCount used = rnd(0, cap);
      if (rnd(0, 3) == 0) used = cap - (cap - used) / 2 * 2;  // create ties
      if (rnd(0, 4) == 0) used = 0;
      s.pool.allocate({{i, used}});
    }
    const bool use_override = rnd(0, 1) == 1;
    for (InstanceId id : inst) {
      TokenCount f = use_override ? rnd(0, cap) : s.pool.at(id).kv_free();
      free_ov.push_back(f);
      tot_free += f;
    }
    const int nreq = static_cast<int>(rnd(1, 4));
    PrefillPlan plan;
    plan.instances = inst;
    TokenCount budget = std::max<TokenCount>(tot_free, 1);
    std::vector<TokenCount> lens;
    for (int r = 0; r < nreq; ++r) {
      Request req;
      req.id = r;
      req.input_len = rnd(1, std::max<TokenCount>(1, budget / nreq));
      if (rnd(0, 9) == 0) req.input_len = budget + 1;  // infeasible case
      lens.push_back(req.input_len);
      s.requests.push_back(req);
    }
    std::vector<RequestId> order(nreq);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](RequestId a, RequestId b) {
      return lens[a] > lens[b];
    });
    plan.requests = order;
    json free_now = json::array();
    for (InstanceId id : inst) free_now.push_back(s.pool.at(id).kv_free());
    json j{{"fn", "plan_prefill_scale_down"}, {"instances", inst},
           {"free", free_now}, {"free_override", use_override ? json(free_ov) : json::array()},
           {"requests", order}, {"input_lens", lens}};
    try {
      if (use_override) {
        plan_prefill_scale_down(s, plan, free_ov);
      } else {
        plan_prefill_scale_down(s, plan, {});
      }
      json pl = json::object();
      for (const auto& [rid, p] : plan.placement) pl[std::to_string(rid)] = placement_json(p);
      j["ok"] = true;
      j["decode_instances"] = plan.decode_instances;
      j["placement"] = pl;
      j["ring_volume"] = plan.ring_volume;
    } catch (const InfeasiblePlanError&) {
      j["ok"] = false;
      j["error"] = "InfeasiblePlanError";
    }
    out << j.dump() << "\n";
  }

  // plan_decode_step_core.
  Sib sib = load_default_sib(ref);
  for (int t = 0; t < 300; ++t) {
    const int m = static_cast<int>(rnd(1, 8));
    std::vector<InstanceId> all(m);
    std::iota(all.begin(), all.end(), 0);
    std::shuffle(all.begin(), all.end(), rng);
    const int d = static_cast<int>(rnd(1, m));
    std::vector<InstanceId> members(all.begin(), all.begin() + d);
    std::sort(members.begin(), members.end());
    std::vector<InstanceId> idle(all.begin() + d, all.end());
    if (rnd(0, 1)) std::sort(idle.begin(), idle.end());
    std::map<InstanceId, TokenCount> free;
    json free_j = json::object();
    for (int i = 0; i < m; ++i) {
      free[i] = rnd(0, 3) == 0 ? rnd(0, 3) : rnd(0, 200);
      free_j[std::to_string(i)] = free[i];
    }
    const int b = static_cast<int>(rnd(0, 3) == 0 ? rnd(60, 200) : rnd(0, 40));
    std::vector<RequestId> batch(b);
    std::iota(batch.begin(), batch.end(), 100);
    SchedulerParams sp;
    sp.enable_scale_up = rnd(0, 4) != 0;
    std::vector<InstanceId> idle_in = idle;
    GroupScalePlan plan =
        plan_decode_step_core(members, batch, free, idle, sib, sp, 7);
    out << json{{"fn", "plan_decode_step_core"}, {"members", members},
                {"batch_size", b}, {"free", free_j}, {"idle", idle_in},
                {"enable_scale_up", sp.enable_scale_up}, {"threshold", 64},
                {"max_dop", 8}, {"feasible", plan.feasible},
                {"masters", plan.step.masters},
                {"add_instances", plan.step.add_instances},
                {"idle_after", idle}}
               .dump()
        << "\n";
  }

  // assign_masters + decode_step_comm.
  for (int t = 0; t < 200; ++t) {
    const int m = static_cast<int>(rnd(1, 8));
    KvPool pool(m, 50);
    for (int i = 0; i < m; ++i) pool.allocate({{i, rnd(0, 50)}});
    std::vector<InstanceId> ids(m);
    std::iota(ids.begin(), ids.end(), 0);
    std::shuffle(ids.begin(), ids.end(), rng);
    const int k = static_cast<int>(rnd(1, m));
    std::vector<InstanceId> masters(ids.begin(), ids.begin() + k);
    const int b = static_cast<int>(rnd(0, 40));
    std::vector<RequestId> batch;
    for (int r = 0; r < b; ++r) batch.push_back(rnd(0, 1000));
    std::sort(batch.begin(), batch.end());
    batch.erase(std::unique(batch.begin(), batch.end()), batch.end());
    std::shuffle(batch.begin(), batch.end(), rng);
    MasterAssignment a = assign_masters(batch, masters);
    ParallelGroup g;
    g.instances = ids;
    std::sort(g.instances.begin(), g.instances.end());
    g.masters = masters;
    DecodeCommResult c = decode_step_comm(g, a, pool);
    json aj = json::object();
    for (const auto& [mm, rs] : a) aj[std::to_string(mm)] = rs;
    json app = json::object();
    for (const auto& [r, mm] : c.append_at) app[std::to_string(r)] = mm;
    json fr = json::array();
    for (int i = 0; i < m; ++i) fr.push_back(pool.at(i).kv_free());
    out << json{{"fn", "assign_masters+decode_step_comm"}, {"batch", batch},
                {"masters", masters}, {"group", g.instances}, {"free", fr},
                {"assignment", aj}, {"ok", c.ok}, {"full_master", c.full_master},
                {"query_volume", c.query_volume},
                {"overlappable_volume", c.overlappable_volume}, {"append_at", app}}
               .dump()
        << "\n";
  }

  // build_ring_schedule / coverage / volume, and proactive_scale_down.
  for (int t = 0; t < 100; ++t) {
    const int d = static_cast<int>(rnd(1, 16));
    std::vector<InstanceId> group(d);
    std::iota(group.begin(), group.end(), 0);
    std::shuffle(group.begin(), group.end(), rng);
    std::vector<TokenCount> seg;
    for (int i = 0; i < d; ++i) seg.push_back(rnd(0, 1000));
    RingSchedule ring = build_ring_schedule(group, seg);
    json rounds = json::array();
    for (const auto& rd : ring.rounds) {
      json rj = json::array();
      for (const RingTransfer& tr : rd) rj.push_back({tr.from, tr.to, tr.volume});
      rounds.push_back(rj);
    }
    KvPool pool(16, 20000);
    for (int i = 0; i < 16; ++i) pool.allocate({{i, rnd(0, 20000)}});
    ScaleDownPlan sd;
    sd.source_instances = group;
    const int ns = static_cast<int>(rnd(1, d));
    sd.target_instances.assign(group.begin(), group.begin() + ns);
    TokenCount total = std::accumulate(seg.begin(), seg.end(), TokenCount{0});
    KvPlacement pl;
    TokenCount left = total;
    for (int i = 0; i < ns; ++i) {
      TokenCount share = i == ns - 1 ? left : rnd(0, left);
      if (share > 0) pl[sd.target_instances[i]] = share;
      left -= share;
    }
    if (rnd(0, 9) == 0 && !pl.empty()) pl.begin()->second += 1;  // count mismatch
    sd.target[0] = pl;
    json fr = json::array();
    for (int i = 0; i < 16; ++i) fr.push_back(pool.at(i).kv_free());
    json j{{"fn", "ring+proactive_scale_down"}, {"group", group}, {"segments", seg},
           {"rounds", rounds}, {"total_comm_volume", ring.total_comm_volume()},
           {"coverage", ring.coverage()}, {"targets", sd.target_instances},
           {"target_placement", placement_json(pl)}, {"free", fr}};
    try {
      ScaleDownResult r = proactive_scale_down(ring, sd, pool);
      j["ok"] = true;
      j["extra_migration_volume"] = r.extra_migration_volume;
      j["transient_buffer_tokens"] = r.transient_buffer_tokens;
    } catch (const InfeasiblePlanError&) {
      j["ok"] = false;
    }
    out << j.dump() << "\n";
  }

  // reactive_migrate.
  for (int t = 0; t < 200; ++t) {
    const int m = static_cast<int>(rnd(1, 8));
    KvPool pool(m, 1000);
    for (int i = 0; i < m; ++i) pool.allocate({{i, rnd(0, 1000)}});
    std::vector<InstanceId> src(m);
    std::iota(src.begin(), src.end(), 0);
    std::shuffle(src.begin(), src.end(), rng);
    src.resize(static_cast<size_t>(rnd(1, m)));
    std::vector<InstanceId> tgt(src.begin(), src.begin() + rnd(1, static_cast<int64_t>(src.size())));
    TokenCount total = rnd(0, 2000);
    ReactiveMigrateResult r = reactive_migrate(pool, src, tgt, total);
    json fr = json::array();
    for (int i = 0; i < m; ++i) fr.push_back(pool.at(i).kv_free());
    out << json{{"fn", "reactive_migrate"}, {"sources", src}, {"targets", tgt},
                {"total", total}, {"free", fr}, {"feasible", r.feasible},
                {"blocked_instance", r.blocked_instance},
                {"per_source_headroom", r.per_source_headroom},
                {"final_placement", placement_json(r.final_placement)},
                {"migration_volume", r.migration_volume}}
               .dump()
        << "\n";
  }

  // Cost model evaluation on the default SIB.
  for (int t = 0; t < 100; ++t) {
    const int d = static_cast<int>(rnd(1, 8));
    std::vector<TokenCount> lens;
    for (int r = 0, n = static_cast<int>(rnd(1, 5)); r < n; ++r) lens.push_back(rnd(1, 500000));
    const int b = static_cast<int>(rnd(0, 200));
    const TokenCount resident = rnd(0, 4000000);
    const int k = static_cast<int>(rnd(1, 8));
    out << json{{"fn", "sib"}, {"dop", d}, {"lengths", lens},
                {"prefill_ms", sib.prefill_time(lens, {d, 1})}, {"batch", b},
                {"resident", resident}, {"masters", k},
                {"decode_ms", sib.decode_time(b, resident, {d, 1}, k)}}
               .dump()
        << "\n";
  }
  ModelConfig tiny{2, 512, 8, 2, 524288};
  ModelConfig lwm;
  out << json{{"fn", "kv_bytes_per_token"}, {"tiny", kv_bytes_per_token(tiny)},
              {"lwm7b", kv_bytes_per_token(lwm)}}
             .dump()
      << "\n";
  std::cout << "mechanics_random.jsonl written\n";
}

}  // namespace

// Seeded small traces on a tight tiny cluster; the first one whose run
// contains both a preemption drain (MigrationPlan, engine.cpp:260-309) and a
// displaced-KV move (resolve_foreign_kv, engine.cpp:587-648) is recorded.
struct PreemptCase {
  int instances = 0;
  TokenCount capacity = 0;
  std::vector<TraceRecord> trace;
};

PreemptCase find_preempting_trace(const std::string& ref) {
  ModelConfig tiny{2, 512, 8, 2, 524288};
  for (uint64_t seed = 1; seed < 20000; ++seed) {
    std::mt19937_64 rng(seed);
    const int m = 4 + static_cast<int>(rng() % 5);
    const TokenCount cap = 1000 + static_cast<TokenCount>(rng() % 4000);
    std::vector<TraceRecord> tr;
    const int n = 6 + static_cast<int>(rng() % 10);
    double t = 0;
    for (int i = 0; i < n; ++i) {
      t += static_cast<double>(rng() % 300);
      tr.push_back({t, 100 + static_cast<TokenCount>(rng() % (2 * cap)),
                    1 + static_cast<TokenCount>(rng() % 120)});
    }
    EngineParams params;
    params.exact_output_reservation = true;
    Engine eng(KvPool(m, cap), tiny, load_default_sib(ref), make_policy(parse_policy("esp")),
               params);
    eng.submit(tr);
    try {
      eng.run();
    } catch (const SimError&) {
      continue;
    }
    int drains = 0, displaced = 0;
    for (const Event& e : eng.log().events()) {
      if (e.kind == EventKind::kMigration && e.detail == "displaced") ++displaced;
      if (e.kind == EventKind::kMigration && e.detail.rfind("drop=", 0) == 0) ++drains;
    }
    if (drains > 0 || displaced > 0) {
      std::cout << "preempting trace: seed " << seed << ", " << m << " x " << cap << ", "
                << drains << " drains, " << displaced << " displaced moves\n";
      return {m, cap, tr};
    }
  }
  std::cout << "no preempting trace found\n";
  return {};
}

int main(int argc, char** argv) {
  if (argc >= 4 && std::string(argv[1]) == "fit") {
    // The measured-SIB loop: B200 ProfileSample records
    // (esp_dump_profiles) -> the reference's own Sib::load / fit_all / save
    // (cost_model.cpp:202-281), i.e. what `espsim fit-sib` does.
    Sib sib = Sib::load(argv[2]);
    sib.fit_all();
    sib.save(argv[3]);
    return 0;
  }
  if (argc < 3) {
    std::cerr << "usage: golden_driver <reference_root> <outdir> | fit <profiles> <out>\n";
    return 2;
  }
  const std::string ref = argv[1], outdir = argv[2];
  mechanics(ref, outdir);

  ModelConfig tiny{2, 512, 8, 2, 524288};
  ModelConfig lwm;  // 32 x 4096, 32 kv heads, bf16
  run_scenario({"config1_tiny", 2, 200000, tiny, "esp", true, {{0, 4096, 64}}}, ref, outdir);
  run_scenario({"config1_tiny_tight", 2, 4096, tiny, "esp", true, {{0, 4096, 64}}}, ref, outdir);
  run_scenario({"tiny_multi", 4, 6000, tiny, "esp", true,
                {{0, 3000, 8}, {0, 1500, 6}, {1, 700, 12}, {2, 2500, 4}, {40, 900, 9},
                 {41, 4100, 5}, {300, 1200, 7}, {301, 300, 3}}},
               ref, outdir);
  run_scenario({"config3_128k", 8, 65600, lwm, "esp", true, {{0, 131072, 2}}}, ref, outdir);
  for (int d : {1, 2, 4, 8}) {
    run_scenario({"config2_32k_d" + std::to_string(d), 8, 300000, lwm,
                  d == 8 ? "static-tp" : "static-hybrid:" + std::to_string(d), true,
                  {{0, 32768, 2}}},
                 ref, outdir);
  }
  run_config4(ref, outdir);
  {
    PreemptCase pc = find_preempting_trace(ref);
    if (!pc.trace.empty()) {
      run_scenario({"tiny_preempt", pc.instances, pc.capacity, tiny, "esp", true, pc.trace}, ref,
                   outdir);
    }
  }
  // the baseline policies on the same data path — chunked
  // prefill (chunks ride on decode steps) and prefill/decode disaggregation
  // (engine-internal "handoff" KV moves, engine.cpp:194-244).
  run_scenario({"tiny_chunked", 2, 20000, tiny, "chunked:512", true,
                {{0, 1500, 6}, {0, 700, 5}, {30, 2100, 4}, {60, 300, 7}, {90, 900, 3}}},
               ref, outdir);
  run_scenario({"tiny_disagg", 2, 20000, tiny, "disagg:1+1", true,
                {{0, 1500, 6}, {0, 700, 5}, {30, 2100, 4}, {60, 300, 7}, {90, 900, 3}}},
               ref, outdir);
  TraceSpec spec;
  spec.distribution = "mixed";
  spec.requests_per_s = 0.5;
  spec.count = 24;
  spec.seed = 7;
  run_scenario({"config5_mixed", 8, 317000, lwm, "esp", false, gen_trace(spec)}, ref, outdir);
  return 0;
}
