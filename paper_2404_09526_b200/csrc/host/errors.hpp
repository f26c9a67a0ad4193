// Error taxonomy of the B200 ESP data path, mapped 1:1 onto the reference's
// (proj/include/espsim/types.hpp:48-109) and onto the C-ABI status codes in
// include/esp_abi.h. Exceptions never cross the ABI (abi.cpp catches them).
#pragma once

#include <stdexcept>
#include <string>

#include "esp_abi.h"

namespace esp {

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

struct ConfigError : Error {
  explicit ConfigError(const std::string& w) : Error(ESP_ERR_CONFIG, w) {}
};
struct InfeasiblePlanError : Error {
  explicit InfeasiblePlanError(const std::string& w) : Error(ESP_ERR_INFEASIBLE, w) {}
};
struct InternalError : Error {
  explicit InternalError(const std::string& w) : Error(ESP_ERR_INTERNAL, w) {}
};
struct CapacityError : Error {  // AllocResult{ok=false, violating}
  CapacityError(int inst, const std::string& w) : Error(ESP_ERR_CAPACITY, w), instance(inst) {}
  int instance;
};
struct MasterFullError : Error {  // DecodeCommResult{ok=false, full_master}
  MasterFullError(int inst, const std::string& w) : Error(ESP_ERR_MASTER_FULL, w), instance(inst) {}
  int instance;
};
struct UnknownStrategyError : Error {
  explicit UnknownStrategyError(const std::string& w) : Error(ESP_ERR_UNKNOWN_STRATEGY, w) {}
};
struct CudaError : Error {
  explicit CudaError(const std::string& w) : Error(ESP_ERR_CUDA, w) {}
};
struct NoDeviceError : Error {
  explicit NoDeviceError(const std::string& w) : Error(ESP_ERR_NO_DEVICE, w) {}
};

}  // namespace esp
