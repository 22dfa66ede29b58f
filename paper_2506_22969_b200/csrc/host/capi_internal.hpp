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

// binary16 runs of slab plans, step by step (device/runtime.cu; used by multi.cu):
// the plan that runs them (null: the run takes the fp32 path), the ring conversion
// at run start, launch t of a run, and the launch counters
sst_plan* plan_h16_runner(sst_plan* p, uint64_t launches);
void plan_h16_begin(sst_plan* hp, int src, void* stream);
void plan_h16_step(sst_plan* hp, int src, uint64_t t, uint64_t launches, void* stream);
uint64_t plan_launches(const sst_plan* p, bool h16);
void plan_add_launches(sst_plan* p, uint64_t launches, uint64_t h16);

}  // namespace sstc
