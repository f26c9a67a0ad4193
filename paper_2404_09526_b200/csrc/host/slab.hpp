// Lazily backed KV slab of one elastic instance: [layer][slot][hidden] bf16.
//
// The instance's full logical capacity (ElasticInstance.kv_capacity, which
// must equal the reference's for counter parity) is reserved as virtual
// address space with the CUDA VMM API; physical HBM is mapped per layer
// region only up to the highest slot ever handed out (slots are handed out
// lowest-first), in 2 MiB-granular chunks that at least double each time.
// A cluster whose instances are mostly empty (e.g. config 3: 8 instances x
// 65,600 slots, KV resting on 2 survivors) then costs HBM only for resident
// tokens.
//
// Peer access: cudaDeviceEnablePeerAccess does not cover cuMemCreate/cuMemMap
// memory, so every chunk is mapped with one CUmemAccessDesc per device of the
// runtime that can reach the owner (the owner first). The cross-domain paths
// (push prefill into a survivor's slab on another GPU, chunk gathers, KV
// moves) dereference slabs from those devices.
#pragma once

#include <cuda.h>

#include <cstddef>
#include <cstdint>
#include <vector>

namespace esp {

class LazySlab {
 public:
  LazySlab() = default;
  LazySlab(const LazySlab&) = delete;
  LazySlab& operator=(const LazySlab&) = delete;
  ~LazySlab();

  // Reserves layers x capacity rows of row_bytes on `device`; every mapped
  // chunk is read/write for `device` and each of `peers` (devices that
  // access it over NVLink; duplicates and `device` itself are ignored).
  void reserve(int device, int layers, int64_t capacity, size_t row_bytes,
               const std::vector<int>& peers = {});
  // Maps physical memory so rows [0, rows) of every layer are backed.
  void ensure(int64_t rows);

  void* base() const { return reinterpret_cast<void*>(base_); }
  // Element (bf16) distance between consecutive layer regions.
  int64_t layer_stride_elems() const { return static_cast<int64_t>(layer_stride_ / 2); }
  size_t mapped_bytes() const { return mapped_ * static_cast<size_t>(layers_); }
  // Devices granted access (owner first).
  const std::vector<int>& access_devices() const { return access_; }
  // cuMemGetAccess of `device` on every mapped chunk: true iff all of them
  // are read/write for it (false when nothing is mapped yet).
  bool readable_writable_by(int device) const;

 private:
  int device_ = -1;
  std::vector<int> access_;
  int layers_ = 0;
  int64_t capacity_ = 0;
  size_t row_bytes_ = 0;
  size_t gran_ = 0;
  size_t layer_stride_ = 0;
  size_t mapped_ = 0;  // bytes mapped at the start of each layer region
  CUdeviceptr base_ = 0;
  size_t reserved_ = 0;
  struct Chunk {
    CUmemGenericAllocationHandle h;
    CUdeviceptr at;
    size_t bytes;
  };
  std::vector<Chunk> chunks_;
};

}  // namespace esp
