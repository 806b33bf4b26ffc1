// capi_internal.hpp -- what other translation units of the C ABI (comm.cpp)
// may see of the session and batch objects defined in capi.cpp.
#pragma once
#include <mutex>
#include <string>

#include "../../include/hegmm_b200.h"
#include "context.hpp"

namespace hgm {

Context& session_context(hgm_ctx* c);
int session_device(const hgm_ctx* c);
std::recursive_mutex& session_exec_mutex(hgm_ctx* c);
void session_retain(hgm_ctx* c);
void session_release(hgm_ctx* c);
hgm_ctx* batch_session(hgm_batch* b);
const u64* batch_results(const hgm_batch* b, size_t* count);
// records the thread-local message behind hgm_last_error and returns `code`
int set_error(int code, const std::string& msg);
// device (or managed) memory, as opposed to host memory that must be staged
bool is_device_pointer(const void* p);

// Makes a device current for a scope and restores the caller's afterwards.
struct DeviceGuard {
    int prev = -1, want;
    explicit DeviceGuard(int dev) : want(dev) {
        if (want < 0) return;
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != want) cudaSetDevice(want);
    }
    ~DeviceGuard() {
        if (want >= 0 && prev >= 0 && prev != want) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

}  // namespace hgm
