// Shared helpers between the compile-tier (capi_compile.cpp) and the device
// tier (device/runtime.cu) of the C ABI: thread-local error text and the
// exception -> sst_status mapping.
#pragma once

#include <stdexcept>
#include <string>

#include "sparstencil.h"

namespace sstc {

struct CudaError : std::runtime_error {
    bool no_device = false;
    CudaError(const std::string& msg, bool nodev) : std::runtime_error(msg), no_device(nodev) {}
};

void set_error(const std::string& msg);
sst_status from_current_exception();  // call inside a catch block

}  // namespace sstc
