// Seeded synthetic weights (random init, no checkpoint exists offline).
// Every element is a pure function of (seed, tensor, layer, logical row,
// logical col): a splitmix64 hash feeding a 4-term Irwin-Hall sum scaled to
// N(0, 0.02^2). All arithmetic before the final single multiply is exact, so
// the CPU oracle (oracle/llama_ref.c, which restates this definition) and the
// device produce bit-identical bf16 weights.
#pragma once

#include <cstdint>

#ifndef ESP_HD
#ifdef __CUDACC__
#define ESP_HD __host__ __device__
#else
#define ESP_HD
#endif
#endif

namespace esp::k {

enum SyntheticTensor : int {
  kTensorEmbed = 1,
  kTensorQ = 2,
  kTensorK = 3,
  kTensorV = 4,
  kTensorO = 5,
  kTensorGate = 6,
  kTensorUp = 7,
  kTensorDown = 8,
  kTensorLmHead = 9,
};

ESP_HD inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

ESP_HD inline float synthetic_weight(uint64_t seed, int tensor, int layer, int64_t row,
                                     int64_t col, int64_t cols) {
  const uint64_t idx = static_cast<uint64_t>(row) * static_cast<uint64_t>(cols) +
                       static_cast<uint64_t>(col);
  const uint64_t key = (static_cast<uint64_t>(tensor) << 56) ^
                       (static_cast<uint64_t>(layer) << 48) ^ idx;
  const uint64_t h = splitmix64(seed ^ splitmix64(key));
  const int32_t s = static_cast<int32_t>(h & 0xFFFF) + static_cast<int32_t>((h >> 16) & 0xFFFF) +
                    static_cast<int32_t>((h >> 32) & 0xFFFF) + static_cast<int32_t>(h >> 48);
  return static_cast<float>(s - 131070) * 5.2857997e-07f;
}

}  // namespace esp::k
