// Host-side placement mechanics of the ESP hot path — B200-runtime
// restatements of the reference functions that decide where every token's KV
// lives and which instances do what. They run on the host between kernel
// launches, so they are plain C++ over small vectors; each cites the
// reference function it must match bit-for-bit (checked against
// tests/golden/mechanics_random.jsonl, generated from the reference itself).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <utility>
#include <vector>

#include "errors.hpp"

namespace esp {

using InstanceId = int32_t;
using RequestId = int64_t;
using Tokens = int64_t;

// Instance -> token count, ascending instance (reference KvPlacement,
// cluster.hpp:44).
using Placement = std::map<InstanceId, Tokens>;

// (instance, tokens) in the order a request's tokens are laid out.
using FillOrder = std::vector<std::pair<InstanceId, Tokens>>;

int64_t kv_bytes_per_token(int layers, int hidden_dim, int kv_heads, int bytes_per_element);

struct PrefillScaleDown {
  std::vector<InstanceId> decode_instances;  // ascending
  std::vector<FillOrder> fill;               // per request, fill order
  Tokens ring_volume = 0;
};

// scheduler.cpp:663-713. free[i] belongs to instances[i].
PrefillScaleDown plan_prefill_scale_down(const std::vector<InstanceId>& instances,
                                         const std::vector<Tokens>& free,
                                         const std::vector<Tokens>& input_lens);

struct SibRecord {
  int dop = 1, tp = 1;
  double alpha_p = 0, beta_p = 0, gamma_p = 0;
  double alpha_d = 0, beta_d = 0, gamma_d = 0;
  int threshold = 64;
  double tipping_ms = 0;
};

class Sib {
 public:
  Sib() = default;
  explicit Sib(std::vector<SibRecord> recs) : recs_(std::move(recs)) {}
  bool has(int dop, int tp) const { return find(dop, tp) != nullptr; }
  const SibRecord& record(int dop, int tp) const;
  double prefill_time_sums(double sum, double sum_sq, int dop, int tp) const;  // cost_model.cpp:169-173
  double decode_time(int b, Tokens resident, int dop, int tp, int k) const;    // cost_model.cpp:175-187

 private:
  const SibRecord* find(int dop, int tp) const;
  std::vector<SibRecord> recs_;
};

struct DecodeStepPlan {
  bool feasible = false;
  std::vector<InstanceId> masters;        // ascending
  std::vector<InstanceId> add_instances;  // scale-up, in take order
};

// scheduler.cpp:726-804; idle_pool is consumed from the front.
DecodeStepPlan plan_decode_step(std::vector<InstanceId> members, int64_t batch_size,
                                const std::map<InstanceId, Tokens>& free,
                                std::vector<InstanceId>& idle_pool, const Sib& sib, int tp,
                                bool enable_scale_up);

// esp_mechanics.cpp:220-238: master -> requests (ascending request ids).
std::map<InstanceId, std::vector<RequestId>> assign_masters(std::vector<RequestId> batch,
                                                            std::vector<InstanceId> masters);

struct DecodeComm {
  Tokens query_volume = 0;
  Tokens overlappable_volume = 0;
};
// esp_mechanics.cpp:240-264; throws MasterFullError on the first master
// (ascending id) lacking room for its appends.
DecodeComm decode_step_comm(int d, const std::map<InstanceId, std::vector<RequestId>>& assign,
                            const std::map<InstanceId, Tokens>& free);

struct RingTransfer {
  InstanceId from, to;
  Tokens volume;
};
struct RingSchedule {
  std::vector<InstanceId> instances;
  std::vector<Tokens> segments;
  std::vector<std::vector<RingTransfer>> rounds;  // d rounds; the last is empty
  Tokens total_comm_volume() const;
  // Origin ring position of the block held by position i in round r.
  static int origin(int i, int r, int d) { return ((i - r) % d + d) % d; }
};
RingSchedule build_ring_schedule(const std::vector<InstanceId>& group,
                                 const std::vector<Tokens>& segments);  // esp_mechanics.cpp:45-70

struct ScaleDownResult {
  Tokens extra_migration_volume = 0;
  Tokens transient_buffer_tokens = 0;
};
// esp_mechanics.cpp:78-136 over the aggregate target placement.
ScaleDownResult proactive_scale_down(const RingSchedule& ring,
                                     const std::vector<InstanceId>& sources,
                                     const std::vector<InstanceId>& targets,
                                     const FillOrder& target_placement,
                                     const std::map<InstanceId, Tokens>& free);

struct ReactiveResult {
  bool feasible = false;
  InstanceId blocked_instance = -1;
  Tokens per_source_headroom = 0;
  Placement final_placement;
  Tokens migration_volume = 0;
};
ReactiveResult reactive_migrate(const std::map<InstanceId, Tokens>& free,
                                const std::vector<InstanceId>& sources,
                                const std::vector<InstanceId>& targets,
                                Tokens total);  // esp_mechanics.cpp:138-218

}  // namespace esp
