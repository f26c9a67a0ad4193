// Placement mechanics of the ESP hot path (see planner.hpp). Every function
// here is pinned bit-exactly to the reference by tests/test_planner_golden.py.
#include "planner.hpp"

#include <algorithm>
#include <numeric>
#include <set>
#include <string>

namespace esp {

int64_t kv_bytes_per_token(int layers, int hidden_dim, int kv_heads, int bytes_per_element) {
  // cluster.cpp:23-34: ModelConfig::validate, then K and V over all layers.
  if (layers <= 0 || hidden_dim <= 0 || kv_heads <= 0 || bytes_per_element <= 0) {
    throw ConfigError("model config fields must be positive");
  }
  return 2LL * layers * hidden_dim * bytes_per_element;
}

// ---- scheduler.cpp:663-713 -------------------------------------------------
PrefillScaleDown plan_prefill_scale_down(const std::vector<InstanceId>& instances,
                                         const std::vector<Tokens>& free,
                                         const std::vector<Tokens>& input_lens) {
  if (instances.size() != free.size()) throw InternalError("one free count per ring instance");
  const Tokens total = std::accumulate(input_lens.begin(), input_lens.end(), Tokens{0});
  std::map<InstanceId, Tokens> room_of;
  for (size_t i = 0; i < instances.size(); ++i) room_of[instances[i]] = free[i];

  // Survivor preference: most free first, lower id on ties.
  std::vector<InstanceId> pref = instances;
  std::sort(pref.begin(), pref.end(), [&](InstanceId a, InstanceId b) {
    return room_of[a] != room_of[b] ? room_of[a] > room_of[b] : a < b;
  });
  // Fewest survivors whose free slots cover the batch.
  Tokens covered = 0;
  size_t n_surv = 0;
  for (; n_surv < pref.size() && covered < total; ++n_surv) covered += room_of[pref[n_surv]];
  if (covered < total) throw InfeasiblePlanError("batch KV exceeds its instance interval");
  n_surv = std::max<size_t>(n_surv, 1);

  PrefillScaleDown out;
  out.decode_instances.assign(pref.begin(), pref.begin() + static_cast<long>(n_surv));
  std::sort(out.decode_instances.begin(), out.decode_instances.end());

  // One cursor over the survivors, shared by the whole batch: request r+1
  // continues on the survivor where request r stopped.
  std::vector<Tokens> room(n_surv);
  for (size_t s = 0; s < n_surv; ++s) room[s] = room_of[pref[s]];
  size_t cur = 0;
  for (Tokens len : input_lens) {
    FillOrder fill;
    for (Tokens left = len; left > 0;) {
      while (cur < n_surv && room[cur] == 0) ++cur;
      if (cur >= n_surv) throw InternalError("scale-down fill overflow");
      const Tokens take = std::min(left, room[cur]);
      fill.emplace_back(pref[cur], take);
      room[cur] -= take;
      left -= take;
    }
    out.fill.push_back(std::move(fill));
  }
  out.ring_volume = (static_cast<Tokens>(instances.size()) - 1) * total;
  return out;
}

// ---- cost_model.cpp:157-187 --------------------------------------------------
const SibRecord* Sib::find(int dop, int tp) const {
  for (const SibRecord& r : recs_) {
    if (r.dop == dop && r.tp == tp) return &r;
  }
  return nullptr;
}

const SibRecord& Sib::record(int dop, int tp) const {
  const SibRecord* r = find(dop, tp);
  if (!r) {
    throw UnknownStrategyError("no timing record for strategy dop=" + std::to_string(dop) +
                               " tp=" + std::to_string(tp));
  }
  return *r;
}

double Sib::prefill_time_sums(double sum, double sum_sq, int dop, int tp) const {
  const SibRecord& c = record(dop, tp);
  return c.alpha_p + c.beta_p * sum + c.gamma_p * sum_sq;
}

double Sib::decode_time(int b, Tokens resident, int dop, int tp, int k) const {
  if (b < 0 || resident < 0 || k < 1) throw InternalError("bad decode_time arguments");
  const SibRecord& c = record(dop, tp);
  double per_request = c.beta_d * b;
  if (b > c.threshold) per_request /= static_cast<double>(k);  // masters share it
  return c.alpha_d + per_request +
         c.gamma_d * static_cast<double>(resident) / static_cast<double>(dop);
}

// ---- scheduler.cpp:726-804 ---------------------------------------------------
DecodeStepPlan plan_decode_step(std::vector<InstanceId> members, int64_t b,
                                const std::map<InstanceId, Tokens>& free,
                                std::vector<InstanceId>& idle_pool, const Sib& sib, int tp,
                                bool enable_scale_up) {
  DecodeStepPlan plan;
  if (b == 0) return plan;
  const int d0 = static_cast<int>(members.size());
  const int64_t thr = sib.has(d0, tp) ? sib.record(d0, tp).threshold : 0;
  const bool past_thr = thr > 0 && b > thr;

  auto grab_idle = [&]() -> std::optional<InstanceId> {
    if (!enable_scale_up || idle_pool.empty() ||
        !sib.has(static_cast<int>(members.size()) + 1, tp)) {
      return std::nullopt;
    }
    const InstanceId id = idle_pool.front();
    idle_pool.erase(idle_pool.begin());
    members.push_back(id);
    plan.add_instances.push_back(id);
    return id;
  };
  const size_t want = past_thr ? static_cast<size_t>((b + thr - 1) / thr) : 0;
  // Compute-bound batches first grow to ceil(b / thr) members.
  while (past_thr && members.size() < want && grab_idle()) {
  }

  auto masters_for = [&](size_t k) -> std::optional<std::vector<InstanceId>> {
    std::vector<InstanceId> pref = members;
    std::sort(pref.begin(), pref.end(), [&](InstanceId x, InstanceId y) {
      const Tokens fx = free.at(x), fy = free.at(y);
      return fx != fy ? fx > fy : x < y;
    });
    if (k > pref.size()) return std::nullopt;
    std::vector<InstanceId> pick(pref.begin(), pref.begin() + static_cast<long>(k));
    std::sort(pick.begin(), pick.end());
    // Balanced request counts, the extra ones on the lowest ids.
    const int64_t base = b / static_cast<int64_t>(k), extra = b % static_cast<int64_t>(k);
    for (size_t i = 0; i < k; ++i) {
      if (free.at(pick[i]) < base + (static_cast<int64_t>(i) < extra ? 1 : 0)) return std::nullopt;
    }
    return pick;
  };

  for (;;) {
    const size_t k0 = past_thr ? std::min(want, members.size()) : 1;
    for (size_t k = k0; k <= members.size(); ++k) {
      if (auto pick = masters_for(k)) {
        plan.feasible = true;
        plan.masters = std::move(*pick);
        return plan;
      }
    }
    if (!grab_idle()) break;  // no reachable master placement: stall
  }
  return plan;
}

// ---- esp_mechanics.cpp:220-238 -------------------------------------------------
std::map<InstanceId, std::vector<RequestId>> assign_masters(std::vector<RequestId> batch,
                                                            std::vector<InstanceId> masters) {
  if (masters.empty()) throw InfeasiblePlanError("no master instances");
  std::sort(batch.begin(), batch.end());
  std::sort(masters.begin(), masters.end());
  std::map<InstanceId, std::vector<RequestId>> out;
  for (InstanceId m : masters) out[m];
  for (RequestId r : batch) {
    InstanceId best = masters.front();
    for (InstanceId m : masters) {
      if (out[m].size() < out[best].size()) best = m;
    }
    out[best].push_back(r);
  }
  return out;
}

// ---- esp_mechanics.cpp:240-264 -------------------------------------------------
DecodeComm decode_step_comm(int d, const std::map<InstanceId, std::vector<RequestId>>& assign,
                            const std::map<InstanceId, Tokens>& free) {
  Tokens b = 0;
  for (const auto& kv : assign) b += static_cast<Tokens>(kv.second.size());
  DecodeComm c;
  c.query_volume = b * (d - 1);
  c.overlappable_volume = b * static_cast<Tokens>(assign.empty() ? 0 : assign.size() - 1);
  for (const auto& [m, reqs] : assign) {
    if (reqs.empty()) continue;
    auto it = free.find(m);
    const Tokens room = it == free.end() ? 0 : it->second;
    if (room < static_cast<Tokens>(reqs.size())) {
      throw MasterFullError(m, "master " + std::to_string(m) +
                                   " cannot hold its appended tokens");
    }
  }
  return c;
}

// ---- esp_mechanics.cpp:24-70 ------------------------------------------------------
Tokens RingSchedule::total_comm_volume() const {
  Tokens t = 0;
  for (const auto& rd : rounds) {
    for (const RingTransfer& x : rd) t += x.volume;
  }
  return t;
}

RingSchedule build_ring_schedule(const std::vector<InstanceId>& group,
                                 const std::vector<Tokens>& segments) {
  if (group.empty()) throw InfeasiblePlanError("ring over an empty group");
  if (group.size() != segments.size()) {
    throw InfeasiblePlanError("one segment size per ring instance required");
  }
  for (Tokens s : segments) {
    if (s < 0) throw InfeasiblePlanError("negative ring segment");
  }
  RingSchedule ring;
  ring.instances = group;
  ring.segments = segments;
  const int d = static_cast<int>(group.size());
  ring.rounds.resize(static_cast<size_t>(d));
  for (int r = 0; r + 1 < d; ++r) {
    for (int i = 0; i < d; ++i) {
      ring.rounds[r].push_back({group[i], group[(i + 1) % d],
                                segments[static_cast<size_t>(RingSchedule::origin(i, r, d))]});
    }
  }
  return ring;
}

// ---- esp_mechanics.cpp:78-136 -------------------------------------------------------
ScaleDownResult proactive_scale_down(const RingSchedule& ring,
                                     const std::vector<InstanceId>& sources,
                                     const std::vector<InstanceId>& targets,
                                     const FillOrder& target_placement,
                                     const std::map<InstanceId, Tokens>& free) {
  const std::set<InstanceId> ring_set(ring.instances.begin(), ring.instances.end());
  bool same = sources.size() == ring_set.size();
  for (InstanceId s : sources) same = same && ring_set.count(s) > 0;
  if (!same) throw InfeasiblePlanError("plan sources disagree with the ring group");
  if (targets.empty()) throw InfeasiblePlanError("plan keeps no target instance");
  if (targets.size() > ring_set.size()) {
    throw InfeasiblePlanError("plan targets exceed the prefill group");
  }
  const std::set<InstanceId> target_set(targets.begin(), targets.end());
  for (InstanceId t : target_set) {
    if (!ring_set.count(t)) {
      throw InfeasiblePlanError("target instance " + std::to_string(t) +
                                " is outside the prefill group");
    }
  }
  // Every block visits every ring member, so any split over the targets is
  // reachable by retention alone; what remains is bookkeeping.
  const Tokens circulated =
      std::accumulate(ring.segments.begin(), ring.segments.end(), Tokens{0});
  Tokens planned = 0;
  for (const auto& [inst, tok] : target_placement) planned += tok;
  if (planned != circulated) {
    throw InfeasiblePlanError("plan retains a different token count than prefilled");
  }
  std::map<InstanceId, Tokens> per_target;
  for (const auto& [inst, tok] : target_placement) {
    if (tok < 0) throw InfeasiblePlanError("negative target share");
    if (tok > 0 && !target_set.count(inst)) {
      throw InfeasiblePlanError("placement lands outside target instances");
    }
    per_target[inst] += tok;
  }
  for (const auto& [inst, tok] : per_target) {
    auto it = free.find(inst);
    if (tok > (it == free.end() ? 0 : it->second)) {
      throw InfeasiblePlanError("target instance " + std::to_string(inst) +
                                " lacks free slots for its share");
    }
  }
  const Tokens d = static_cast<Tokens>(ring.instances.size());
  return ScaleDownResult{0, (circulated + d - 1) / d};
}

// ---- esp_mechanics.cpp:138-218 ------------------------------------------------------
ReactiveResult reactive_migrate(const std::map<InstanceId, Tokens>& free,
                                const std::vector<InstanceId>& sources,
                                const std::vector<InstanceId>& targets, Tokens total) {
  if (sources.empty()) throw InfeasiblePlanError("no source instances");
  if (total < 0) throw InfeasiblePlanError("negative token total");
  const std::set<InstanceId> src_set(sources.begin(), sources.end());
  for (InstanceId t : targets) {
    if (!src_set.count(t)) {
      throw InfeasiblePlanError("reactive targets must survive from the sources");
    }
  }
  auto free_of = [&](InstanceId i) {
    auto it = free.find(i);
    return it == free.end() ? Tokens{0} : it->second;
  };
  ReactiveResult res;
  const Tokens n = static_cast<Tokens>(sources.size());
  const Tokens share = (total + n - 1) / n;
  res.per_source_headroom = share;
  // The even-share prefill needs that headroom on every source up front.
  for (InstanceId s : sources) {
    if (free_of(s) < share) {
      res.blocked_instance = s;
      return res;
    }
  }
  std::map<InstanceId, Tokens> held;
  Tokens left = total;
  for (InstanceId s : sources) {
    held[s] = std::min(share, left);
    left -= held[s];
  }
  if (targets.empty()) throw InfeasiblePlanError("reactive migration keeps no target instance");
  std::vector<InstanceId> pref = targets;
  std::sort(pref.begin(), pref.end(), [&](InstanceId a, InstanceId b) {
    const Tokens fa = free_of(a) - held[a], fb = free_of(b) - held[b];
    return fa != fb ? fa > fb : a < b;
  });
  const std::set<InstanceId> tgt_set(targets.begin(), targets.end());
  Tokens moving = 0;
  for (InstanceId s : sources) {
    if (!tgt_set.count(s)) moving += held[s];
  }
  res.migration_volume = moving;
  std::map<InstanceId, Tokens> final_tok;
  for (InstanceId t : targets) final_tok[t] = held[t];
  for (InstanceId t : pref) {
    if (moving == 0) break;
    const Tokens take = std::min(free_of(t) - final_tok[t], moving);
    if (take > 0) {
      final_tok[t] += take;
      moving -= take;
    }
  }
  if (moving > 0) {
    res.blocked_instance = pref.back();
    return res;
  }
  res.feasible = true;
  for (const auto& [i, t] : final_tok) {
    if (t > 0) res.final_placement[i] = t;
  }
  return res;
}

}  // namespace esp
