// LazySlab: CUDA VMM (cuMemAddressReserve / cuMemCreate / cuMemMap) through
// driver entry points, so the library needs no libcuda link.
#include "slab.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "errors.hpp"

namespace esp {

namespace {

struct Vmm {
  CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*free_va)(CUdeviceptr, size_t);
  CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                     unsigned long long);
  CUresult (*release)(CUmemGenericAllocationHandle);
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                  unsigned long long);
  CUresult (*unmap)(CUdeviceptr, size_t);
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*get_access)(unsigned long long*, const CUmemLocation*, CUdeviceptr);
  CUresult (*granularity)(size_t*, const CUmemAllocationProp*,
                          CUmemAllocationGranularity_flags);
};

template <typename F>
void entry(const char* name, F& fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p) {
    throw CudaError(std::string("driver entry point missing: ") + name);
  }
  fn = reinterpret_cast<F>(p);
}

const Vmm& vmm() {
  static Vmm v = [] {
    Vmm x{};
    entry("cuMemAddressReserve", x.reserve);
    entry("cuMemAddressFree", x.free_va);
    entry("cuMemCreate", x.create);
    entry("cuMemRelease", x.release);
    entry("cuMemMap", x.map);
    entry("cuMemUnmap", x.unmap);
    entry("cuMemSetAccess", x.set_access);
    entry("cuMemGetAccess", x.get_access);
    entry("cuMemGetAllocationGranularity", x.granularity);
    return x;
  }();
  return v;
}

void ok(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + " failed: " + std::to_string(r));
}

CUmemAllocationProp prop_for(int device) {
  CUmemAllocationProp p{};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = device;
  return p;
}

size_t round_up(size_t x, size_t g) { return (x + g - 1) / g * g; }

}  // namespace

void LazySlab::reserve(int device, int layers, int64_t capacity, size_t row_bytes,
                       const std::vector<int>& peers) {
  device_ = device;
  access_.assign(1, device);
  for (int d : peers) {
    if (std::find(access_.begin(), access_.end(), d) == access_.end()) access_.push_back(d);
  }
  layers_ = layers;
  capacity_ = capacity;
  row_bytes_ = row_bytes;
  const CUmemAllocationProp p = prop_for(device);
  ok(vmm().granularity(&gran_, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
  layer_stride_ = round_up(static_cast<size_t>(capacity) * row_bytes, gran_);
  reserved_ = layer_stride_ * static_cast<size_t>(layers);
  ok(vmm().reserve(&base_, reserved_, gran_, 0, 0), "cuMemAddressReserve");
}

void LazySlab::ensure(int64_t rows) {
  const size_t need = std::min(round_up(static_cast<size_t>(rows) * row_bytes_, gran_), layer_stride_);
  if (need <= mapped_) return;
  const size_t target = std::min(layer_stride_, std::max(need, round_up(mapped_ * 2, gran_)));
  const size_t grow = target - mapped_;
  const CUmemAllocationProp p = prop_for(device_);
  std::vector<CUmemAccessDesc> acc(access_.size());
  for (size_t i = 0; i < access_.size(); ++i) {
    acc[i] = CUmemAccessDesc{};
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = access_[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  for (int l = 0; l < layers_; ++l) {
    const CUdeviceptr at = base_ + static_cast<CUdeviceptr>(l) * layer_stride_ + mapped_;
    CUmemGenericAllocationHandle h;
    ok(vmm().create(&h, grow, &p, 0), "cuMemCreate (KV slab)");
    if (vmm().map(at, grow, 0, h, 0) != CUDA_SUCCESS) {
      vmm().release(h);
      throw CudaError("cuMemMap (KV slab) failed");
    }
    chunks_.push_back({h, at, grow});
    ok(vmm().set_access(at, grow, acc.data(), acc.size()), "cuMemSetAccess (KV slab)");
  }
  mapped_ = target;
}

bool LazySlab::readable_writable_by(int device) const {
  if (chunks_.empty()) return false;
  CUmemLocation loc{};
  loc.type = CU_MEM_LOCATION_TYPE_DEVICE;
  loc.id = device;
  for (const Chunk& c : chunks_) {
    unsigned long long flags = 0;
    if (vmm().get_access(&flags, &loc, c.at) != CUDA_SUCCESS ||
        flags != CU_MEM_ACCESS_FLAGS_PROT_READWRITE) {
      return false;
    }
  }
  return true;
}

LazySlab::~LazySlab() {
  if (!base_) return;
  for (const Chunk& c : chunks_) {
    vmm().unmap(c.at, c.bytes);
    vmm().release(c.h);
  }
  vmm().free_va(base_, reserved_);
}

}  // namespace esp
